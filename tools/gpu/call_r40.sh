B="python bench.py --steps 40 --warmup 3 --no-bf16-block --no-cpu-baseline --no-e2e"
for w in 2 1 0; do timeout 900 $B --candidate-warmup $w --json-out gpurun_out/r40_W$w.json > /dev/null 2>&1; python -c "
import json; d=json.load(open('gpurun_out/r40_W$w.json')); print('W=$w', round(d['value']), round(d['ms_per_step']), round(d['roofline']['frac'],3), json.dumps(d['quality_dp_over_10k']), d['tuning_wall_s'])"; done
