timeout 300 python tools/dbg_quick.py c1 > gpurun_out/dbg6.log 2>&1
timeout 300 python tools/dbg_quick.py c2 4000000 >> gpurun_out/dbg6.log 2>&1
