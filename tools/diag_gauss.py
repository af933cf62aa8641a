import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2209_08722_b200 import sketching as S
n, w, seed = 100_000, 40, 42
ref = np.random.Generator(np.random.Philox(seed)).standard_normal((n, w)).ravel() / np.sqrt(w)
got = S.build_gaussian_sketch(n, w, seed).dense.cpu().numpy().ravel()
bad = np.nonzero(got != ref)[0]
print("mismatches", bad.size, "first", bad[:10])
if bad.size:
    i = bad[0]
    print("ref", ref[i-2:i+4] * np.sqrt(w)); print("got", got[i-2:i+4] * np.sqrt(w))
    print("tile guess (draw/4096)", i / 4096)
