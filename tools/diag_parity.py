"""Per-quantity error report of a golden_large case (which tensor carries the error): rotated K / V rows per layer
and first-token logits, relative per element (floor 1e-2 max|ref|) and relative to max|ref|."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_07590_b200 import turbokv as T  # noqa: E402


def errs(got, ref):
    got, ref = np.asarray(got, np.float64).ravel(), np.asarray(ref, np.float64).ravel()
    m = np.abs(ref).max()
    e = np.abs(got - ref)
    return f"per-elem(floor 1%) {float((e / np.maximum(np.abs(ref), 1e-2 * m)).max()):.3e}  max-rel {e.max() / m:.3e}"


def main(name="c2ctx", dtype="f32", flags=0):
    G = os.path.join(ROOT, "tests", "golden")
    meta = json.load(open(os.path.join(G, "golden_large.json")))[name]
    A = np.load(os.path.join(G, "golden_large.npz"))
    eng = T.Engine(T.ModelConfig(**meta["config"]), meta["seed"], dtype=dtype, flags=flags, store_capacity_tokens=1 << 15)
    offs = A[f"{name}.payload_offsets"]
    pays = [A[f"{name}.payloads"][offs[i]:offs[i + 1]] for i in range(len(offs) - 1)]
    ids = eng.ingest_chunks(pays)
    sel = [ids[i] for i in meta["requests"][0]["chunks"]]
    for mode, tag in ((T.PositionMode.Reordered, "reordered"), (T.PositionMode.Composite, "composite")):
        with eng.assemble(sel, mode) as ctx:
            if f"{name}.kv_rows" in A and tag == "reordered":
                rows = A[f"{name}.kv_rows"]
                for layer in range(meta["config"]["layer_num"]):
                    print(name, dtype, "K layer", layer, errs(ctx.read_kv(layer, "k", True)[rows], A[f"{name}.krot{layer}"]))
                    print(name, dtype, "V layer", layer, errs(ctx.read_kv(layer, "v", True)[rows], A[f"{name}.v{layer}"]))
            lg = eng.prefill_query(ctx, A[f"{name}.r0.query"])
            print(name, dtype, tag, "logits", errs(lg, A[f"{name}.r0.{tag}.logits"]))


if __name__ == "__main__":
    main(*sys.argv[1:3], *(int(x) for x in sys.argv[3:]))
