"""The C ABI driven from C (tests/c/abi_smoke.c): a host program with no Python
or torch calls skb_sparse_embedding and skb_normal_apply on cudaMalloc'd
memory; its output is checked against the oracle here."""

import os
import shutil
import subprocess

import numpy as np
import pytest

from conftest import ROOT
from oracle import ipm_oracle as O

pytestmark = pytest.mark.gpu


def test_c_host_program(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    pkg = os.path.join(ROOT, "paper_2209_08722_b200")
    exe = str(tmp_path / "abi_smoke")
    cuda = "/usr/local/cuda"
    subprocess.run(["gcc", "-O2", os.path.join(ROOT, "tests", "c", "abi_smoke.c"),
                    "-I", os.path.join(ROOT, "include"), "-I", f"{cuda}/include",
                    "-L", pkg, "-lskb", "-L", f"{cuda}/lib64", "-lcudart",
                    f"-Wl,-rpath,{pkg}:{cuda}/lib64", "-o", exe], check=True)
    seed = 2024
    k = np.random.SeedSequence(seed).generate_state(2, np.uint64)
    out = subprocess.run([exe, str(int(k[0])), str(int(k[1]))], check=True,
                         capture_output=True, text=True).stdout.split("\n")
    fields = {ln.split()[0]: ln.split()[1:] for ln in out if ln.strip()}
    cols, vals = O.sparse_embedding(1000, 64, 2, seed)
    assert [int(c) for c in fields["cols"]] == cols.reshape(-1)[:8].tolist()
    assert [float(v) for v in fields["vals"]] == vals.reshape(-1)[:8].tolist()
    m, n = 6, 50
    A = np.array([[((i + 2 * j) % 7) - 3.0 for j in range(n)] for i in range(m)])
    d2 = 0.5 + 0.01 * np.arange(n)
    z = 1.0 + np.arange(m)
    ref = A @ (d2 * (A.T @ z))
    u = np.array([float(v) for v in fields["u"]])
    assert np.max(np.abs(u - ref)) <= 1e-13 * np.abs(ref).max()
