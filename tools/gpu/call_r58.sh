timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -1
for e in 0 1; do if [ $e = 1 ]; then export DB200_NO_PDL=1; fi; echo "nopdl=$e"
timeout 300 python tools/time_points.py --layer r18.conv1 9:16,1,256,32,0 9:8,2,64,64,0 2>&1 | grep ns
timeout 300 python tools/time_points.py --layer vgg.3-64@224 --dtype bf16 10:32,1,256,32,1 2>&1 | grep ns
done
