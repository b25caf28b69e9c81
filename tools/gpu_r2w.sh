# r2w: histogram variants (hot-leaf cache / direct atomics / match_any aggregation) on c3 binned and c2 stream
mkdir -p gpurun_out/r2w
V="paper_2005_03156_b200/_lib/var/lib_h1.so paper_2005_03156_b200/_lib/var/lib_h2.so"
EXPV_HIST=1 timeout 900 python tools/exp_variants.py c3 1e9 binned 0 $V > gpurun_out/r2w/c3_hist.log 2>&1
timeout 900 python tools/exp_variants.py c3 1e9 binned 0 > gpurun_out/r2w/c3_nohist.log 2>&1
EXPV_HIST=1 timeout 900 python tools/exp_variants.py c2 1e8 stream 0 $V > gpurun_out/r2w/c2_hist.log 2>&1
timeout 900 python tools/exp_variants.py c2 1e8 stream 0 > gpurun_out/r2w/c2_nohist.log 2>&1
