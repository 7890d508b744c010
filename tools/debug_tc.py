"""Diagnose the tcgen05 GEMM operand-major variants on small shapes."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1708_02983_b200 import _lib  # noqa: E402
from paper_1708_02983_b200.device import stream_ptr  # noqa: E402


def run(m, n, k, a_major, b_major, precision=3, batch=1):
    rng = np.random.default_rng(0)
    A = rng.integers(-3, 4, (batch, m, k)).astype(np.float32)
    B = rng.integers(-3, 4, (batch, n, k)).astype(np.float32)
    As = np.ascontiguousarray(A.transpose(0, 2, 1)) if a_major else A
    Bs = np.ascontiguousarray(B.transpose(0, 2, 1)) if b_major else B
    lda = m if a_major else k
    ldb = n if b_major else k
    Ad, Bd = torch.from_numpy(As).cuda(), torch.from_numpy(Bs).cuda()
    Cd = torch.full((batch, m, n), -777.0, device="cuda")
    d = _lib.TcGemmDesc(m, n, k, batch, Ad.data_ptr(), lda, m * k, Bd.data_ptr(), ldb, n * k,
                        Cd.data_ptr(), n, 1, m * n, None, 0, None, 0, 0, 0, 0, 0, precision,
                        a_major, b_major, None, 0)
    rc = _lib.load().esgd_tc_gemm_f32(C.byref(d), stream_ptr())
    torch.cuda.synchronize()
    ref = np.einsum("zmk,znk->zmn", A.astype(np.float64), B.astype(np.float64))
    got = Cd.cpu().numpy()
    err = np.abs(got - ref).max()
    print(f"m={m} n={n} k={k} a_major={a_major} b_major={b_major} prec={precision} rc={rc} maxerr={err:.3g}"
          f" zeros={np.mean(got == 0):.2f} sentinel={np.mean(got == -777):.2f}")
    if err > 1e-3:
        # is it a transpose / permutation of the right answer?
        g, r = got[0], ref[0]
        print("  got[0,:8]", g[0, :8])
        print("  ref[0,:8]", r[0, :8])
        for name, cand in (("A^T-ish", None),):
            pass
    return err


if __name__ == "__main__":
    for am, bm in ((0, 0), (0, 1), (1, 0), (1, 1)):
        for prec in (1, 3):
            run(128, 64, 32, am, bm, prec)
            run(128, 128, 64, am, bm, prec)
