import ctypes as C, sys
sys.path.insert(0, ".")
from paper_2410_07590_b200 import turbokv as T
L = T.lib()
# (M, N, K, splits, swiglu) ; splits chosen per cps
for knobs in [(4, 110, 2, 1), (4, 110, 1, 1), (3, 80, 1, 1), (6, 150, 1, 1), (8, 200, 1, 1)]:
    T._check(L.tkv_debug_set_gemm_knobs(*knobs))
    cps = knobs[2]
    shapes = {"qkv": (64, 4608, 3584, 8 if cps == 2 else 4), "o": (64, 3584, 3584, 10 if cps == 2 else 5),
              "down": (64, 3584, 18944, 10 if cps == 2 else 5)}
    out = []
    for name, (M, N, K, sp) in shapes.items():
        ms = C.c_double()
        T._check(L.tkv_debug_gemm_bench(0, M, N, K, sp, 0, 50, C.byref(ms)))
        out.append(f"{name} {ms.value*1e3:6.2f} us ({N*K*2/(ms.value/1e3)/1e9:5.0f} GB/s)")
    print(knobs, " | ".join(out), flush=True)
