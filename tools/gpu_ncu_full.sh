# one full ncu capture of the projection kernel (after a clean plain run)
CFG=${1:-c2}
PTS=${2:-20000000}
TAG=${3:-r1}
python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu --no-e2e --points $PTS > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:project_kernel -s 1 -c 1 \
    -o gpurun_out/prof_$TAG python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu --no-e2e --points $PTS > gpurun_out/ncu_$TAG.log 2>&1
echo ncu_rc=$?
