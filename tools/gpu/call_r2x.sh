B="python bench.py --steps 40 --warmup 3 --no-bf16-block --no-cpu-baseline --no-e2e"
timeout 900 $B --json-out gpurun_out/r2x_v0.json > /dev/null 2>gpurun_out/r2x_v0.err
timeout 900 $B --droplet-policy radius --json-out gpurun_out/r2x_v1.json > /dev/null 2>gpurun_out/r2x_v1.err
timeout 900 $B --evolve-pop 32 --evolve-elite 8 --json-out gpurun_out/r2x_v2.json > /dev/null 2>gpurun_out/r2x_v2.err
timeout 900 $B --droplet-policy radius --droplet-sketch-factor 3 --json-out gpurun_out/r2x_v3.json > /dev/null 2>gpurun_out/r2x_v3.err
for v in 0 1 2 3; do python -c "
import json; d=json.load(open('gpurun_out/r2x_v$v.json')); print('v$v', json.dumps(d['quality_dp_over_10k']), d['tuning_wall_s'], round(d['roofline']['frac'],3))"; done
