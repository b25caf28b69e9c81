# r2ab: bulk-copy (TMA) staging variant of the binned query vs default; hist defaults
mkdir -p gpurun_out/r2ab
timeout 900 python tools/exp_variants.py c3 1e9 binned 0 paper_2005_03156_b200/_lib/var/lib_bulk.so > gpurun_out/r2ab/c3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"binned_query" --csv --log-file gpurun_out/r2ab/launches.csv \
  python tools/exp_variants.py c3 1e9 binned 0 paper_2005_03156_b200/_lib/var/lib_bulk.so > gpurun_out/r2ab/ncu.log 2>&1
timeout 900 python tools/exp_variants.py c4 2e8 binned 0 paper_2005_03156_b200/_lib/var/lib_bulk.so > gpurun_out/r2ab/c4.log 2>&1
timeout 900 python bench.py --config c2 --hist --no-cpu --no-e2e > gpurun_out/r2ab/c2_hist.log 2>&1
timeout 900 python bench.py --config c5 --steps 3 --no-cpu --no-e2e --check-points 2000000 > gpurun_out/r2ab/c5.log 2>&1
