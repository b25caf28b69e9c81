# A/B of the default library vs _lib/var variants (c2 sweep, two passes),
# then (PROF=1) launch list + one full capture of stream_kernel (default lib)
TAG=${1:-ab}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
if [ -n "$TESTS" ]; then
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest=$? >> gpurun_out/${TAG}_pytest.log
fi
for pass in 1 2; do
timeout 400 python tools/exp_sweep.py ${SWEEP_MS:-0} >> gpurun_out/${TAG}_sweep.log 2>&1
if [ -n "$QUICK" ]; then FASTMAP_B200_QUICK=1 SWEEP_LIB_TAG=quick timeout 400 python tools/exp_sweep.py ${SWEEP_MS:-0} >> gpurun_out/${TAG}_sweep.log 2>&1; fi
for v in paper_2005_03156_b200/_lib/var/*.so; do
  FASTMAP_B200_LIB=$v timeout 400 python tools/exp_sweep.py ${SWEEP_MS:-0} >> gpurun_out/${TAG}_sweep.log 2>&1
done
done
if [ -n "$PROF" ]; then
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
timeout 300 $CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"stream_kernel|resolve_kernel|resolve_quick_kernel" --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncul.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KER:-stream_kernel} -s 3 -c 1 \
  -o gpurun_out/${TAG}_prof $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo ncu=$? >> gpurun_out/${TAG}_ncu.log
fi
