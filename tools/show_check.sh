# summarize a gpu_check.sh run
TAG=${1:-chk}
tail -3 gpurun_out/${TAG}_pytest.log
for f in c2 c4 c1 approx; do
  grep -h '^{' gpurun_out/${TAG}_bench_$f.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); i=d['config']['index']
    print('$f', round(d['ms_per_step'],4), '%.3g'%d['value'], d['parity'], i['nx'], i['ny'], i.get('query_block_log2'), d['config']['index_build_s'])"
done
