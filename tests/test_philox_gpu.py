"""Library pin of the oracle's Philox4x32-10 against cuRAND's device implementation
(curand_Philox4x32_10, /usr/local/cuda/include/curand_philox4x32_x.h), reading C15."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_oracle_philox_matches_curand(tmp_path, oracle_mod):
    import torch
    so = str(tmp_path / "ref.so")
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                           "-Xcompiler", "-fPIC", "-o", so, os.path.join(HERE, "cuda", "curand_philox_ref.cu")])
    lib = C.CDLL(so)
    rng = np.random.default_rng(42)
    n = 20000
    ctr = rng.integers(0, 2 ** 32, (n, 4), dtype=np.uint64).astype(np.uint32)
    ctr[:100] = 0
    ctr[100:200, 0] = np.arange(100)
    key = rng.integers(0, 2 ** 32, (n, 2), dtype=np.uint64).astype(np.uint32)
    tc = torch.from_numpy(ctr.view(np.int32)).cuda()
    tk = torch.from_numpy(key.view(np.int32)).cuda()
    to = torch.zeros((n, 4), dtype=torch.int32, device="cuda")
    assert lib.curand_philox_ref(C.c_void_p(tc.data_ptr()), C.c_void_p(tk.data_ptr()), C.c_void_p(to.data_ptr()), n) == 0
    ref = to.cpu().numpy().view(np.uint32)
    for i in range(n):
        assert np.array_equal(oracle_mod.philox(ctr[i], key[i]), ref[i]), i
