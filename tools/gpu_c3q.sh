# quick c3 query check (200M points) after gpu_check.sh
timeout 2400 python bench.py --config c3 --points 200000000 --no-cpu --no-e2e --steps 5 > gpurun_out/c3q_bench.log 2>&1; echo rc=$? >> gpurun_out/c3q_bench.log
