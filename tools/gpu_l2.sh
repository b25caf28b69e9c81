mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_l2.log 2>&1; echo pytest=$? >> gpurun_out/pytest_l2.log
timeout 300 python tools/exp_sweep.py 0 14 20 > gpurun_out/l2_on.log 2>&1
FASTMAP_B200_L2_PERSIST=0 timeout 300 python tools/exp_sweep.py 0 > gpurun_out/l2_off.log 2>&1
python -c "
import torch; p=torch.cuda.get_device_properties(0); print('persistingL2CacheMaxSize', getattr(p,'persisting_l2_cache_max_size',None), 'L2', p.L2_cache_size)" >> gpurun_out/l2_on.log 2>&1
