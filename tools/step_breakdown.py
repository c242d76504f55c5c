"""Per-kernel breakdown of the LAST turbo step in an ncu launch list (bench.py --turbo-only).

With --share-json PATH it also writes the per-class share of that step (profiles/launch_share.json), which
bench.py scales to its measured ms_per_step: ncu replays kernels serialised and cold, so only the SHARE of the
step transfers to the real (PDL-overlapped, warm) step, not the absolute times."""
import collections
import csv
import json
import re
import sys

CLASSES = [("gemm", r"gemm_tc_kernel|gemm_mlp_kernel|gemm_simt"), ("attention", r"attn_"),
           ("gather_rope", r"gather_rope"),
           ("epilogue", r"residual_kernel|qkv_epilogue|swiglu|embed_kernel|reduce_splits"), ("other", r".")]


def cls_of(name):
    return next(c for c, rx in CLASSES if re.search(rx, name))


def main(path, share_json=None):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    data = [(r[ki], float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-3)) for r in rows[hi + 1:] if len(r) > vi]
    g = [i for i, (n, _) in enumerate(data) if "gather_rope" in n][-1]
    step = data[g:]
    agg = collections.defaultdict(lambda: [0, 0.0])
    per_cls = collections.defaultdict(float)
    for n, t in step:
        m = re.search(r"(\w+_kernel)(<[^>]*>)?", n)
        k = m.group(1) + (m.group(2) or "") if m else n[:30]
        k = k.replace("__nv_bfloat16", "bf16")
        agg[k][0] += 1
        agg[k][1] += t
        per_cls[cls_of(n)] += t
    tot = sum(v[1] for v in agg.values())
    print(f"one turbo step: {len(step)} launches, {tot / 1000:.3f} ms summed (serialized ncu replay, cold caches)")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {k:40s} {c:4d} {t:9.1f} us {100 * t / tot:5.1f}%")
    if share_json:
        with open(share_json, "w") as f:
            json.dump({"source": path.split("/")[-1], "launches": len(step), "summed_us": tot,
                       "classes": {c: v / tot for c, v in sorted(per_cls.items())}}, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
