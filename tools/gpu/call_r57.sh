timeout 900 python -m pytest tests/test_gpu_dwconv.py -x -q 2>&1 | tail -1
for i in 1 2; do
DB200_NO_PDL=1 timeout 900 python tools/sweep.py --models mobilenetv2,efficientnetb0 --ops depthwise_conv2d --baseline 2000 --out gpurun_out/r57_nopdl$i.jsonl > /dev/null 2>&1
timeout 900 python tools/sweep.py --models mobilenetv2,efficientnetb0 --ops depthwise_conv2d --baseline 2000 --out gpurun_out/r57_pdl$i.jsonl > /dev/null 2>&1
done
for f in nopdl1 pdl1 nopdl2 pdl2; do python -c "
import json
rows=[json.loads(l) for l in open('gpurun_out/r57_$f.jsonl')]
S=[r for r in rows if r.get('summary')]
print('$f', [(s['model'], round(s['model_us_dpansor'],1)) for s in S])"; done
