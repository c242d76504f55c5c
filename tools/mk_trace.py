"""Timeline of one layer-kernel launch (TUNING build, TKV_MK_TRACE=<layer>): per phase, when the CTAs got past its
dependency (A-producer / workers) and finished it, relative to the earliest worker start (us; min / median / max)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import c2_step  # noqa: E402
from paper_2410_07590_b200 import turbokv as T  # noqa: E402

NAMES = ["O", "res1", "gate/up", "down", "res2", "QKV", "qkv-epi"]


def main():
    eng_holder = {}
    orig = T.Engine.__init__

    def keep(self, *a, **k):
        orig(self, *a, **k)
        eng_holder["e"] = self
    T.Engine.__init__ = keep
    c2_step.main(steps=3, flags=128)
    e = eng_holder["e"]
    buf = np.zeros(4096 * 32, np.uint64)
    T._check(T.lib().tkv_debug_mk_trace(e._h, buf.ctypes.data_as(C.POINTER(C.c_uint64)), buf.size))
    tr = buf.reshape(4096, 32)
    tr = tr[tr[:, 0] > 0].astype(np.float64)
    t0 = tr[:, 0].min()
    print(f"{len(tr)} CTAs; worker start spread {(tr[:, 0].max() - t0) / 1e3:.2f} us")
    for p, nm in enumerate(NAMES):
        for slot, what in ((8 + p, "A past dep"), (16 + p, "workers past dep"), (1 + p, "phase done")):
            v = tr[:, slot]
            v = v[v > 0]
            if len(v):
                v = (v - t0) / 1e3
                print(f"  {nm:8s} {what:17s} min {v.min():8.2f}  med {np.median(v):8.2f}  max {v.max():8.2f}")


if __name__ == "__main__":
    main()
