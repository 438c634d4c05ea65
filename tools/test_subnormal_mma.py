"""Does tcgen05.mma kind::f16 keep fp16 / bf16 subnormal A operands exact?  (tools only)
A = raw bit patterns 0..15 (fp16 subnormals l * 2^-24), B = random fp16 weights; compare with fp64."""
import ctypes as C, os, subprocess, sys
import numpy as np
import torch
HERE = os.path.dirname(os.path.abspath(__file__))
so = "/tmp/tc_probe_sub.so"
subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-shared",
                       "-Xcompiler", "-fPIC", "-std=c++17", "-o", so, os.path.join(HERE, "..", "tests", "cuda", "tc_probe.cu")])
P = C.CDLL(so)
g = torch.Generator().manual_seed(1)
for mode, dt in ((1, torch.float16), (2, torch.float16), (0, torch.bfloat16)):
    K, N = 256, 256
    lv = torch.randint(0, 16, (128, K), generator=g, dtype=torch.int16)
    A = lv.view(dt).cuda()                                    # subnormals l * 2^-24 (fp16) / l * 2^-133 (bf16)
    Bf = torch.randn((N, K), generator=g) * 0.05
    B = Bf.to(dt).cuda()
    D = torch.zeros((128, N), dtype=torch.int32, device="cuda")
    rc = P.tc_probe(mode, C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()), C.c_void_p(D.data_ptr()), N, K)
    Dg = D.view(torch.float32).double().cpu()
    ref = A.double().cpu() @ B.double().cpu().T
    scale = A.double().abs().cpu() @ B.double().abs().cpu().T
    err = ((Dg - ref).abs() / scale.clamp_min(1e-300)).max().item()
    print(f"mode {mode} {dt}: rc {rc}  max |ref| {ref.abs().max().item():.3e}  max rel err {err:.3e}  "
          f"zeros in result {int((Dg == 0).sum())}")
