# r2l: scatter-kernel experiments (variant libraries on one c3 index, binned, 162 tiles)
mkdir -p gpurun_out/r2l
V=$(ls paper_2005_03156_b200/_lib/var/*.so)
timeout 1200 python tools/exp_variants.py c3 1e9 binned 64e6 $V > gpurun_out/r2l/var.log 2>&1; echo rc=$? >> gpurun_out/r2l/var.log
