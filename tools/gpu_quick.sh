# quick-record A/B: GPU tests, then c2 sweeps (resolutions) for the default
# library, the variants under _lib/var (lib_head.so = the last commit)
TAG=${1:-q}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
if [ -z "$NO_TESTS" ]; then
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest=$? >> gpurun_out/${TAG}_pytest.log
fi
for pass in 1 2; do
timeout 400 python tools/exp_sweep.py ${SWEEP_MS:-0 12} >> gpurun_out/${TAG}_sweep.log 2>&1
for v in paper_2005_03156_b200/_lib/var/*.so; do
  FASTMAP_B200_LIB=$v timeout 400 python tools/exp_sweep.py ${SWEEP_MS:-0 12} >> gpurun_out/${TAG}_sweep.log 2>&1
done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv >> gpurun_out/${TAG}_smi.txt 2>&1
done
