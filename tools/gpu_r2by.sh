# r2by: compute-sanitizer (memcheck, racecheck) over the binned-path GPU tests
mkdir -p gpurun_out/r2by
timeout 1800 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_binned.py -x -q > gpurun_out/r2by/memcheck.log 2>&1; echo rc=$? >> gpurun_out/r2by/memcheck.log
timeout 2400 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_binned.py -x -q -k "not c3 and not full" > gpurun_out/r2by/racecheck.log 2>&1; echo rc=$? >> gpurun_out/r2by/racecheck.log
