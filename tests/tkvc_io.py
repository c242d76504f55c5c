"""TEST INFRASTRUCTURE: write reference TKVC chunk files (proj/docs/formats.md:114-140,
proj/src/kvstore.cpp:78-132) from oracle K/V so the GPU engine can import exactly the bytes the
reference store would hold. Pinned byte-for-byte against the reference's own CacheStore::store
in tests/test_tkvc_io.py."""
from __future__ import annotations

import os
import struct

import numpy as np


def tkvc_bytes(chunk_id: int, fingerprint: int, k: np.ndarray, v: np.ndarray, kv_head_num: int, head_size: int,
               f32: bool = False) -> bytes:
    L, n, kvd = k.shape
    elem = 4 if f32 else 8
    tb = n * kvd * elem
    out = bytearray(b"TKVC")
    out += struct.pack("<IIIIII", 1, 2 if f32 else 1, L, kv_head_num, head_size, n)
    out += struct.pack("<QQ", fingerprint, chunk_id)
    cur = 44 + L * 16
    for _ in range(L):
        out += struct.pack("<QQ", cur, cur + tb)
        cur += 2 * tb
    dt = "<f4" if f32 else "<f8"
    for layer in range(L):
        out += np.ascontiguousarray(k[layer], dtype=dt).tobytes()
        out += np.ascontiguousarray(v[layer], dtype=dt).tobytes()
    return bytes(out)


def write_tkvc(root: str, chunk_id: int, fingerprint: int, k, v, kv_head_num: int, head_size: int,
               f32: bool = False) -> str:
    path = os.path.join(root, f"{chunk_id:016x}.tkvc")
    with open(path, "wb") as f:
        f.write(tkvc_bytes(chunk_id, fingerprint, k, v, kv_head_num, head_size, f32))
    return path
