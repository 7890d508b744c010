"""Read off the TMA swizzle of a 32x32 fp32 box (SW128 vs SW128_ATOM_32B):
for every element (row k, col m) of the source, print where it lands.

    nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o /tmp/probe_swizzle.so tools/probe_swizzle.cu
    python tools/probe_swizzle.py
"""
import ctypes as C

import torch

lib = C.CDLL("/tmp/probe_swizzle.so")
src = torch.arange(1024, dtype=torch.float32, device="cuda")  # value = k*32 + m
for atom32 in (0, 1):
    out = torch.zeros(1024, device="cuda")
    rc = lib.probe_swizzle(C.c_void_p(out.data_ptr()), C.c_void_p(src.data_ptr()), atom32)
    assert rc == 0, rc
    o = out.cpu().numpy().astype(int)
    pos = {int(v): i for i, v in enumerate(o)}
    ok_formula = True
    for k in range(32):
        for m in range(32):
            byte = pos[k * 32 + m] * 4
            if atom32:
                pred = k * 128 + ((((m * 4) >> 5) ^ (k & 3)) << 5) + ((m * 4) & 31)
            else:
                pred = k * 128 + ((((m * 4) >> 4) ^ (k & 7)) << 4) + ((m * 4) & 15)
            ok_formula &= (byte == pred)
    print("atom32" if atom32 else "sw128", "formula matches:", ok_formula)
    if not ok_formula:
        for k in range(8):
            print("  k", k, [(pos[k * 32 + m] - k * 32) // 8 for m in range(0, 32, 8)])
    print(" row0:", [pos[0 * 32 + m] for m in range(0, 32, 4)], " row1:", [pos[1 * 32 + m] for m in range(0, 32, 4)],
          " row2:", [pos[2 * 32 + m] for m in range(0, 32, 4)])
