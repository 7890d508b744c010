"""Role timeline of the tcgen05 GEMM on CTA 0 (clock64 stamps from a probe
build compiled with -DESGD_TRACE, loaded through ESGD_LIB):

    ESGD_LIB=paper_1708_02983_b200/libesgd_trace.so python tools/trace_gemm.py conv2.fwd

Per K block g: TMA issue (producer), full (split warps start), split done,
MMA issue; per K chunk c: MMA acquires the accumulator buffer, chunk complete
(drain starts), drained. Prints steady-state averages in cycles.
"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import bench_gemm  # noqa: E402
from paper_1708_02983_b200 import _lib  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "conv2.fwd"
    torch.cuda.set_device(0)
    if name.startswith("implicit:"):  # implicit-GEMM conv layer[:pass], e.g. implicit:conv4:fwd
        import bench_conv_gemm
        parts = name.split(":")
        sys.argv = [sys.argv[0], "--only", parts[1]] + (["--pass", parts[2]] if len(parts) > 2 else [])
        bench_conv_gemm.main()  # the last launch is traced
    else:
        shape = next(s for s in bench_gemm.SHAPES if s[0] == name)
        bench_gemm.run(*shape, int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 3, reps=1)
    lib = _lib.load()
    lib.esgd_trace_copy.restype = C.c_int
    buf = np.zeros((8, 4096), dtype=np.uint64)
    assert lib.esgd_trace_copy(C.c_void_p(buf.ctypes.data)) == 0
    t = buf.astype(np.int64)
    tma, mma, acq, full, split, cdone, drained = t[0], t[1], t[2], t[3], t[4], t[5], t[6]
    G = int(np.argmax(mma == 0)) if (mma == 0).any() else 4096
    NC = int(np.argmax(cdone == 0)) if (cdone == 0).any() else 4096
    lo, hi = min(8, G // 4), G - 1
    g = np.arange(lo, hi)
    d = lambda a: float(np.mean(a)) if len(a) else float("nan")
    print(f"{name}: CTA 0 ran {G} K blocks, {NC} chunks")
    print(f"  MMA issue interval per K block     {d(np.diff(mma[lo:hi])):8.0f} cycles")
    print(f"  split work (full -> split done)    {d(split[g] - full[g]):8.0f}")
    print(f"  MMA waits after split done         {d(mma[g] - split[g]):8.0f}")
    print(f"  TMA issue -> data landed (full)    {d(full[g] - tma[g]):8.0f}")
    print(f"  split done of g vs MMA issue g-1   {d(split[g] - mma[g - 1]):8.0f}")
    c = np.arange(min(4, NC // 4), NC - 1)
    print(f"  chunk complete interval            {d(np.diff(cdone[c[0]:c[-1] + 1])):8.0f}")
    print(f"  drain time (complete -> drained)   {d(drained[c] - cdone[c]):8.0f}")
    print(f"  MMA acquires buffer after drained  {d(acq[c[2:]] - drained[c[2:] - 2]) if len(c) > 2 else float('nan'):8.0f}")
    if "--raw" in sys.argv:  # per-K-block stamps (relative to the first TMA issue), first 64 K blocks
        t0 = tma[0]
        for i in range(min(64, G)):
            print(f"    g={i:3d} tma {tma[i] - t0:8d} full {full[i] - t0:8d} split {split[i] - t0:8d} mma {mma[i] - t0:8d}")
        for i in range(min(24, NC)):
            print(f"    c={i:3d} acq {acq[i] - t0:8d} done {cdone[i] - t0:8d} drained {drained[i] - t0:8d}")


if __name__ == "__main__":
    main()
