B="python bench.py --steps 40 --warmup 3 --no-bf16-block --no-cpu-baseline --no-e2e"
for wn in 20000 10000 6000; do DB200_WINDOW_NS=$wn timeout 900 $B --json-out gpurun_out/r41_win$wn.json > /dev/null 2>&1; python -c "
import json; d=json.load(open('gpurun_out/r41_win$wn.json')); print('win=$wn', round(d['value']), round(d['ms_per_step']), round(d['roofline']['frac'],3), json.dumps(d['quality_dp_over_10k']), d['tuning_wall_s'])"; done
