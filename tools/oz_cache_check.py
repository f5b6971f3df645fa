import os, sys
sys.path.insert(0, os.getcwd())
import torch
sys.path.insert(0, "tests")
from synth import dags
from gpu_helpers import run_gpu
w = dags.config_c5(N=256, Lt=8, n_pairs=40, n_trees=120, n_corr=4)
ctx, roots, corr, st, ex = run_gpu(w, flags=64, arena_mb=4096, device_leaves=True)
torch.cuda.synchronize()
print("n_contr", st["n_contr"])
