import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, ctypes as C
import paper_2604_12625_b200 as n
out = np.zeros((128, 24), np.uint32)
print(n._lib.ndgi_debug_tmem_f16_probe(out.ctypes.data_as(C.c_void_p)))
for lane in (0, 1, 37, 127):
    w = out[lane, :16]
    pk = out[lane, 16:]
    print(" packed", [f"{a:.4f}" for a in pk.view(np.uint16).view(np.float16)[:12]])
    lo = (w & 0xffff).astype(np.uint16).view(np.float16)
    hi = (w >> 16).astype(np.uint16).view(np.float16)
    print(lane, [f"{a:.4f}/{b:.4f}" for a, b in zip(lo[:10], hi[:10])])
