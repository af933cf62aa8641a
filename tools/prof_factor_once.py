"""One CholeskyQR2 factor build at (PROF_M, PROF_W) between cudaProfilerStart/Stop
(run under ncu --profile-from-start off for a per-kernel launch list)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2209_08722_b200.kernels import DeviceMatrix
from paper_2209_08722_b200 import preconditioning as PC
m, w = int(os.environ.get("PROF_M", 10000)), int(os.environ.get("PROF_W", 40000))
g = torch.Generator(device="cuda"); g.manual_seed(0)
X = DeviceMatrix(torch.randn((w, m + (m & 1)), dtype=torch.float64, device="cuda", generator=g), m)
PC.build_preconditioner(X); torch.cuda.synchronize()
torch.cuda.profiler.start()
PC.build_preconditioner(X); torch.cuda.synchronize()
torch.cuda.profiler.stop()
