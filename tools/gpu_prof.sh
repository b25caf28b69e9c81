# launch list + full capture of one kernel (after a clean plain run of the same command)
TAG=${1:-p}
KER=${2:-resolve_kernel}
PTS=${3:-20000000}
CFG=${4:-c2}
mkdir -p gpurun_out
CMD="python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu --no-e2e --points $PTS"
timeout 300 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"stream_kernel|resolve_kernel" --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_l_$TAG.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$KER -s 1 -c 1 \
  -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo rc=$?
