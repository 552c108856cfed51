"""Which LBO/SBO make MN-major SWIZZLE_128B bf16 tiles correct (tma.cu).
A wrong guess can fault the context, so every candidate runs in its own
process:  python tools/tma_mn_probe.py [lbo sbo N]"""
import subprocess
import sys

sys.path.insert(0, ".")
if len(sys.argv) == 4:
    import torch
    from paper_2303_01778_b200._lib import lib, ptr
    lbo, sbo, N = map(int, sys.argv[1:])
    K = 128
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.randn(K, 128, device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn(K, N, device="cuda", generator=g).to(torch.bfloat16)
    ref = A.double().t() @ B.double()
    D = torch.zeros(128, N, device="cuda")
    lib.check(lib.pb_tma_bf16_mn_selftest(ptr(A), ptr(B), ptr(D), N, K, lbo, sbo, 0))
    torch.cuda.synchronize()
    print(f"N={N} lbo={lbo} sbo={sbo}: rel err {float((D.double() - ref).norm() / ref.norm()):.2e}", flush=True)
else:
    for N in (64, 128):
        for lbo, sbo in ((1024, 8192), (8192, 1024), (16, 1024), (1024, 1024), (8192, 8192)):
            r = subprocess.run([sys.executable, __file__, str(lbo), str(sbo), str(N)], capture_output=True,
                               text=True, timeout=120)
            out = (r.stdout.strip().splitlines() or ["-"])[-1]
            print(out if r.returncode == 0 else f"N={N} lbo={lbo} sbo={sbo}: FAULT", flush=True)
