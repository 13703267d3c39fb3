python -m paper_2605_04263_b200.build
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for c in qwen3_235b qwen3_8b; do
timeout 600 python bench.py --config $c --steps 40 --warmup 10 --no-cpu-baseline --no-e2e --no-readout --no-naive --no-ragged --no-fp8 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('== $c', 'step %.4f attn %.4f plan %.4f frac %.4f kfrac %.4f' % (d['ms_per_step'], r['attn_ms'], r['kernel_ms_plan'], r['frac'], r['frac_kernel_only']), d['clocks'])"
done
