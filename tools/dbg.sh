SWEEP_MS="0" bash tools/gpu_ab.sh ab23
