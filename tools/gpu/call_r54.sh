timeout 1500 python bench.py --workload vgg_alexnet --steps 14 --warmup 2 --no-cpu-baseline --no-e2e --no-bf16-block --json-out gpurun_out/j_vgg_alexnet_bf16.json > /dev/null 2> gpurun_out/j_vgg.err
timeout 900 python bench.py --workload bert --steps 6 --warmup 2 --no-cpu-baseline --no-e2e --no-bf16-block --json-out gpurun_out/j_bert_bf16.json > /dev/null 2> gpurun_out/j_bert.err
for f in j_vgg_alexnet_bf16 j_bert_bf16; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); print('$f', round(d['value']), round(d['roofline']['frac'],3), json.dumps(d['quality_dp_over_10k']), d['tuning_wall_s'])"; done
