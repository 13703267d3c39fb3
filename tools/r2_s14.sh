TRACE_SAVE=gpurun_out/trace_1s.npy PARSE_LIB=$PWD/paper_2605_04263_b200/libparse_trace1.so timeout 300 python tools/trace_attn.py --config qwen3_235b --batch 4 --show 4 > gpurun_out/trace_1s.txt 2>&1
