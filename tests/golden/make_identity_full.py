"""Reference model identity (weights_checksum / model_fingerprint, proj/src/model.cpp:94-118) of the FULL-SIZE
presets the bench runs (BASELINE configs[1] Qwen2-7B shape, configs[3] Llama-3-8B shape), seed 42.

Materialising these models in f64 takes 52-60 GB, so the checksum is streamed by the oracle restatement
(oracle/tkv_oracle.c:tko_weights_checksum_stream), which tests/test_oracle.py pins against the unmodified
reference's weights_checksum at every size the reference can materialise here. ~1-2 min per model, one core.
Run here:  python tests/golden/make_identity_full.py  ->  tests/golden/identity_full.json
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402

LLAMA3_8B = O.Cfg(32, 32, 8, 128, 4096, 14336, 259, 500000.0, 1e-5)


def main():
    O.build(ref=False)
    out = {}
    for name, cfg in (("qwen2-7b", O.QWEN2_7B), ("llama3-8b", LLAMA3_8B)):
        t = time.time()
        ck, fp = O.Port.stream_identity(cfg, 42)
        out[name] = {"seed": 42, "config": cfg.__dict__, "checksum": f"{ck:016x}", "fingerprint": f"{fp:016x}"}
        print(name, out[name], f"{time.time() - t:.0f}s", flush=True)
    with open(os.path.join(HERE, "identity_full.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
