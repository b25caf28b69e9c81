CMD="python bench.py --config c4 --points 100000000 --steps 2 --warmup 3 --no-cpu --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"stream_kernel|resolve_kernel" --csv --log-file gpurun_out/l_c4.csv $CMD > gpurun_out/l_c4.log 2>&1
python - <<'PY' > gpurun_out/c4_counters.log 2>&1
import sys, torch
sys.path.insert(0, '.')
from paper_2005_03156_b200 import fastmap, synth
cfg = synth.config('c4'); soup = cfg.make_soup(); pts = torch.from_numpy(cfg.make_points(20_000_000, soup=soup)).cuda()
idx = fastmap.build_index(soup, device=0); print(idx.stats())
c = torch.zeros(4, dtype=torch.int64, device='cuda'); idx.project(pts, counters=c); torch.cuda.synchronize(); print(c.tolist())
PY
