timeout 1500 python bench.py --workload vgg_alexnet --steps 14 --warmup 2 --no-cpu-baseline --no-e2e --no-bf16-block --json-out gpurun_out/r2w_vgg_alexnet_bf16.json > gpurun_out/r2w_vgg_alexnet_bf16.line 2> gpurun_out/r2w_vgg.err
timeout 900 python bench.py --workload bert --steps 6 --warmup 2 --no-cpu-baseline --no-e2e --no-bf16-block --json-out gpurun_out/r2w_bert_bf16.json > gpurun_out/r2w_bert_bf16.line 2> gpurun_out/r2w_bert.err
tail -c 400 gpurun_out/r2w_vgg_alexnet_bf16.line; tail -c 400 gpurun_out/r2w_bert_bf16.line
