"""Summarise ncu reports into profiles/ (text + JSON).  Usage:
   python tools/ncu_summary.py <report.ncu-rep> <label> [algorithmic_flops | algorithmic_bytes=N]"""
import csv, io, json, subprocess, sys

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "sm__cycles_elapsed.avg.per_second",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def main():
    rep, label = sys.argv[1], sys.argv[2]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, vals = rows[0], rows[1], rows[2]
    d = {"label": label, "kernel": vals[h.index("Kernel Name")]}
    for k in KEYS:
        if k in h:
            i = h.index(k)
            d[k] = vals[i].replace(",", "") + (" " + units[i] if units[i] else "")
    txt = "\n".join(f"{k:75s} {v}" for k, v in d.items())
    print(txt)
    with open(f"profiles/{label}.txt", "w") as f:
        f.write(f"# ncu --set full --clock-control none summary ({rep})\n" + txt + "\n")


if __name__ == "__main__":
    main()
