"""The AlexNet GEMM shapes through our 3xTF32 tcgen05 GEMM vs cuBLAS via
torch.matmul: fp32 (SGEMM, allow_tf32 off — the same fp32-grade result
class) and plain TF32 (allow_tf32 on — ~1e-3 relative, fails the parity
gate; an upper reference only). Also the relative error of each against an
fp64 product.

    python tools/vs_cublas.py
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import bench_gemm  # noqa: E402


def t_matmul(a, b, reps=10):
    for _ in range(3):
        a @ b
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        a @ b
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def relerr(x, ref):
    return float((x.double() - ref).norm() / ref.norm())


def main():
    torch.cuda.set_device(0)
    print(f"{'shape':12s} {'ours 3xTF32':>12s} {'cuBLAS fp32':>12s} {'cuBLAS tf32':>12s}   (ms; rel err vs fp64: ours / fp32 / tf32)")
    tot = [0.0, 0.0, 0.0]
    for name, m, n, k, am, bm, cm in bench_gemm.SHAPES:
        if name.startswith("x."):
            continue
        t_ours = bench_gemm.run(name, m, n, k, am, bm, cm, 3)
        a = torch.randn(m, k, device="cuda")
        b = torch.randn(k, n, device="cuda")
        torch.backends.cuda.matmul.allow_tf32 = False
        t32 = t_matmul(a, b)
        c32 = a @ b
        torch.backends.cuda.matmul.allow_tf32 = True
        ttf = t_matmul(a, b)
        ctf = a @ b
        torch.backends.cuda.matmul.allow_tf32 = False
        # error of ours on the same operands (row-major A, B; C row-major)
        from paper_1708_02983_b200 import _lib
        from paper_1708_02983_b200.device import stream_ptr
        import ctypes as C
        co = torch.empty(m, n, device="cuda")
        ws = torch.zeros(1 << 24, device="cuda")  # (split-K tile counters start at zero)
        if k % 4 == 0 and n % 4 == 0:
            d = _lib.TcGemmDesc(m, n, k, 1, a.data_ptr(), k, 0, b.data_ptr(), n, 0, co.data_ptr(), n, 1, 0,
                                None, 0, None, 0, 0, 0, 0, 0, 3, 0, 1, ws.data_ptr(), ws.numel())
            _lib.check(_lib.load().esgd_tc_gemm_f32(C.byref(d), stream_ptr()))
            torch.cuda.synchronize()
            ref = a.double() @ b.double()
            errs = f"{relerr(co, ref):.1e} / {relerr(c32, ref):.1e} / {relerr(ctf, ref):.1e}"
        else:
            errs = "-"
        print(f"{name:12s} {t_ours * 1e3:12.3f} {t32 * 1e3:12.3f} {ttf * 1e3:12.3f}   {errs}")
        tot[0] += t_ours; tot[1] += t32; tot[2] += ttf
        del a, b, c32, ctf, co
    print(f"{'total':12s} {tot[0] * 1e3:12.3f} {tot[1] * 1e3:12.3f} {tot[2] * 1e3:12.3f}")


if __name__ == "__main__":
    main()
