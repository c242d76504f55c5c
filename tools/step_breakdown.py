"""Per-kernel breakdown of the LAST turbo step in an ncu launch list (bench.py --turbo-only)."""
import collections
import csv
import re
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    data = [(r[ki], float(r[vi].replace(",", "")) / 1000) for r in rows[hi + 1:] if len(r) > vi]
    g = [i for i, (n, _) in enumerate(data) if "gather_rope" in n][-1]
    step = data[g:]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, t in step:
        m = re.search(r"(\w+_kernel)(<[^>]*>)?", n)
        k = m.group(1) + (m.group(2) or "") if m else n[:30]
        k = k.replace("__nv_bfloat16", "bf16")
        agg[k][0] += 1
        agg[k][1] += t
    tot = sum(v[1] for v in agg.values())
    print(f"one turbo step: {len(step)} launches, {tot / 1000:.3f} ms summed (serialized ncu replay, cold caches)")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {k:40s} {c:4d} {t:9.1f} us {100 * t / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
