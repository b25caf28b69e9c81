# r2x: c3 histogram cost (ncu on the binned query with / without hist), build phase breakdown
mkdir -p gpurun_out/r2x
EXPV_HIST=1 timeout 900 ncu --set full --clock-control none -k regex:"binned_query|widen" -c 2 -o gpurun_out/r2x/prof_hist python tools/exp_variants.py c3 1e9 binned 0 > gpurun_out/r2x/ncu_hist.log 2>&1
timeout 600 python -c "
import sys, json, time
sys.path.insert(0, '.')
from paper_2005_03156_b200 import fastmap, synth
for name in ['c3', 'c4', 'c2']:
    soup = synth.config(name).make_soup()
    t = time.time(); idx = fastmap.build_index(soup, device=0); t = time.time() - t
    st = idx.stats()
    print(json.dumps({'config': name, 'build_s': round(t, 2), 'phase_s': [round(x, 2) for x in st['build_phase_seconds']], 'build_seconds': st['build_seconds'], 'slots_double': st['slots_double'], 'cells_split': st['cells_split'], 'slots_total': st['slots_total']}), flush=True)
    idx.close()
" > gpurun_out/r2x/build.log 2>&1
