CMD="python bench.py --mode simple --config c3s --points 20000000 --steps 2 --warmup 3 --no-cpu --no-e2e"
timeout 600 $CMD > gpurun_out/simple_plain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:simple_kernel -s 3 -c 1 -o gpurun_out/simple_prof $CMD > gpurun_out/simple_ncu.log 2>&1
echo ncu=$? >> gpurun_out/simple_ncu.log
