# r2y: phase-1 double slots on both builders (build identity, parity, c3 full), build times; hist variant h3
mkdir -p gpurun_out/r2y
timeout 1800 python -m pytest tests/test_gpu_build.py tests/test_gpu_parity.py tests/test_gpu_binned.py tests/test_gpu_margin.py tests/test_gpu_c3_full.py tests/test_gpu_approx.py tests/test_gpu_io.py -x -q > gpurun_out/r2y/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2y/pytest.log
timeout 600 python -c "
import sys, json, time
sys.path.insert(0, '.')
from paper_2005_03156_b200 import fastmap, synth
for name in ['c3', 'c4', 'c2']:
    soup = synth.config(name).make_soup()
    t = time.time(); idx = fastmap.build_index(soup, device=0); t = time.time() - t
    st = idx.stats()
    print(json.dumps({'config': name, 'build_s': round(t, 2), 'phase_s': [round(x, 2) for x in st['build_phase_seconds']], 'build_seconds': st['build_seconds'], 'slots_double': st['slots_double'], 'cells_split': st['cells_split'], 'slots_total': st['slots_total'], 'slots_phase1': st['slots_phase1'], 'arena': st['arena_bytes']}), flush=True)
    idx.close()
" > gpurun_out/r2y/build.log 2>&1
V="paper_2005_03156_b200/_lib/var/lib_h3.so paper_2005_03156_b200/_lib/var/lib_h1.so"
EXPV_HIST=1 timeout 900 python tools/exp_variants.py c3 1e9 binned 0 $V > gpurun_out/r2y/c3_hist.log 2>&1
EXPV_HIST=1 timeout 900 python tools/exp_variants.py c2 1e8 stream 0 $V > gpurun_out/r2y/c2_hist.log 2>&1
timeout 900 python tools/exp_binned.py c3 1e9 64e6 > gpurun_out/r2y/c3.log 2>&1
