"""tcgen05 building blocks (descriptors, SS / TS forms, kind::f16 and kind::i8) against torch,
and the accuracy of fp32 accumulation in the tensor core (sizes the float-path error budget)."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def probe(tmp_path_factory):
    so = str(tmp_path_factory.mktemp("tc") / "probe.so")
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-shared",
                           "-Xcompiler", "-fPIC", "-std=c++17", "-DMLPV_WAIT_TIMEOUT=4000000000", "-o", so, os.path.join(HERE, "cuda", "tc_probe.cu")])
    return C.CDLL(so)


def _run(probe, mode, A, B, N, K):
    import torch
    D = torch.zeros((128, N), dtype=torch.int32, device="cuda")
    rc = probe.tc_probe(mode, C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()), C.c_void_p(D.data_ptr()), N, K)
    assert rc == 0, rc
    return D


@pytest.mark.parametrize("mode,N,K", [(0, 256, 64), (0, 256, 256), (0, 16, 128), (1, 128, 256), (2, 256, 128),
                                      (3, 256, 256), (2, 16, 64)])
def test_f16_bf16(probe, mode, N, K):
    import torch
    g = torch.Generator(device="cpu").manual_seed(mode * 1000 + N + K)
    dt = torch.bfloat16 if mode in (0, 3) else torch.float16
    A = torch.randn((128, K), generator=g).to(dt).cuda()
    B = (torch.randn((N, K), generator=g) * 0.1).to(dt).cuda()
    D = _run(probe, mode, A, B, N, K).view(torch.float32).double().cpu()
    ref = A.double().cpu() @ B.double().cpu().T
    scale = (A.double().abs().cpu() @ B.double().abs().cpu().T)
    err = (D - ref).abs() / scale.clamp_min(1e-30)
    assert float(err.max()) < 2e-6, float(err.max())


@pytest.mark.parametrize("mode,N,K", [(4, 256, 128), (4, 32, 64 * 2), (5, 256, 256), (5, 16, 128)])
def test_int8(probe, mode, N, K):
    import torch
    g = torch.Generator(device="cpu").manual_seed(N + K)
    A = torch.randint(0, 256, (128, K), generator=g, dtype=torch.int32).to(torch.uint8).cuda()
    B = torch.randint(-127, 128, (N, K), generator=g, dtype=torch.int32).to(torch.int8).cuda()
    D = _run(probe, mode, A, B, N, K).cpu().long()
    ref = A.cpu().long() @ B.cpu().long().T
    assert torch.equal(D, ref)


def test_fp32_accumulation_error(probe):
    """Float-path error budget: sum of K=784-like exact bf16 products in TMEM fp32 vs fp64."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(7)
    K, N = 256, 256
    A = torch.rand((128, K), generator=g).to(torch.bfloat16).cuda()
    B = (torch.randn((N, K), generator=g) * (2.0 / 784) ** 0.5).to(torch.bfloat16).cuda()
    D = _run(probe, 0, A, B, N, K).view(torch.float32).double().cpu()
    ref = A.double().cpu() @ B.double().cpu().T
    abs_err = (D - ref).abs()
    print(f"tcgen05 bf16 K={K}: max abs err {float(abs_err.max()):.3e}, rms {float(abs_err.pow(2).mean().sqrt()):.3e}, "
          f"|ref| rms {float(ref.pow(2).mean().sqrt()):.3e}")
    assert float(abs_err.max()) < 1e-5


@pytest.fixture(scope="module")
def probe2(tmp_path_factory):
    so = str(tmp_path_factory.mktemp("tc2") / "probe2.so")
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-shared",
                           "-Xcompiler", "-fPIC", "-std=c++17", "-DMLPV_WAIT_TIMEOUT=4000000000", "-o", so,
                           os.path.join(HERE, "cuda", "tc_probe2.cu")])
    return C.CDLL(so)


@pytest.mark.parametrize("mode,N,K", [(0, 256, 128), (0, 32, 64), (1, 256, 256), (1, 64, 128)])
def test_cta_pair_mma(probe2, mode, N, K):
    """cta_group::2: M = 256 split over a CTA pair, B split by N, commit multicast to both CTAs."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(11 + mode + N + K)
    A = torch.randn((256, K), generator=g).to(torch.bfloat16).cuda()
    B = (torch.randn((N, K), generator=g) * 0.1).to(torch.bfloat16).cuda()
    D = torch.zeros((256, N), dtype=torch.int32, device="cuda")
    rc = probe2.tc_probe2(mode, C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()), C.c_void_p(D.data_ptr()), N, K)
    assert rc == 0, rc
    D = D.view(torch.float32).double().cpu()
    ref = A.double().cpu() @ B.double().cpu().T
    scale = A.double().abs().cpu() @ B.double().abs().cpu().T
    assert float(((D - ref).abs() / scale.clamp_min(1e-30)).max()) < 2e-6
