B="python bench.py --steps 40 --warmup 3 --no-bf16-block --no-cpu-baseline --no-e2e"
for ec in 4 3 2; do timeout 900 $B --early-cut $ec --json-out gpurun_out/r44_ec$ec.json > /dev/null 2>&1; python -c "
import json; d=json.load(open('gpurun_out/r44_ec$ec.json')); print('ec=$ec', round(d['value']), round(d['ms_per_step']), round(d['roofline']['frac'],3), d['early_cut_frac'], json.dumps(d['quality_dp_over_10k']), d['tuning_wall_s'])"; done
