timeout 900 python -m pytest tests/test_evolve_parity.py tests/test_gpu_kernels.py -x -q 2>&1 | tail -1
B="python bench.py --steps 40 --warmup 3 --no-bf16-block --no-cpu-baseline --no-e2e"
for i in 1 2 3; do timeout 900 $B --json-out gpurun_out/r52_lin$i.json > /dev/null 2>&1; python -c "
import json; d=json.load(open('gpurun_out/r52_lin$i.json')); print('lineage run $i', round(d['value']), round(d['roofline']['frac'],3), json.dumps(d['quality_dp_over_10k']), d['tuning_wall_s'])"; done
