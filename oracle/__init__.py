"""TEST INFRASTRUCTURE ONLY — ctypes access to the two CPU oracles.

* ``Port``  : oracle/build/libtkv_oracle.so — our float64 C restatement of the
  reference (oracle/tkv_oracle.c). Always buildable (``make -C oracle restatement``).
* ``Ref``   : oracle/_ref/libturbokv_ref.so — the UNMODIFIED reference sources from
  /root/reference/proj/src compiled in place plus the extern-C shim
  oracle/ref_capi.cpp. Built only where /root/reference exists; the built .so
  travels to the GPU box with the snapshot.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package, and only as the checker or the timed CPU baseline.
The product path (paper_2410_07590_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "build", "libtkv_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libturbokv_ref.so")
REF_SRC = "/root/reference/proj"

I64P = C.POINTER(C.c_int64)
I32P = C.POINTER(C.c_int32)
U64P = C.POINTER(C.c_uint64)
F64P = C.POINTER(C.c_double)
U8P = C.POINTER(C.c_uint8)


class OracleCfg(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("layer_num", "head_num", "kv_head_num", "head_size",
                                          "hidden_size", "intermediate_size", "vocab_size")] + \
               [("rope_base", C.c_double), ("norm_eps", C.c_double)]


@dataclass
class Cfg:
    layer_num: int
    head_num: int
    kv_head_num: int
    head_size: int
    hidden_size: int
    intermediate_size: int
    vocab_size: int = 259
    rope_base: float = 10000.0
    norm_eps: float = 1e-6

    def c(self) -> OracleCfg:
        return OracleCfg(self.layer_num, self.head_num, self.kv_head_num, self.head_size,
                         self.hidden_size, self.intermediate_size, self.vocab_size,
                         self.rope_base, self.norm_eps)

    @property
    def kv_dim(self) -> int:
        return self.kv_head_num * self.head_size


# proj/src/config.cpp:44-66
TOY = Cfg(4, 8, 2, 8, 64, 192, 259)
QWEN2_7B = Cfg(28, 28, 4, 128, 3584, 18944, 259)


def qwen_layers(n: int) -> Cfg:
    """Exact Qwen2-7B dims with `n` layers (parity at exact dims, 1-2 layers)."""
    return Cfg(n, 28, 4, 128, 3584, 18944, 259)


def ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def build(ref: bool = True) -> None:
    targets = ["restatement"] + (["ref"] if ref and os.path.isdir(REF_SRC) else [])
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def frame(payload) -> np.ndarray:
    """tok::frame_chunk (proj/src/tokenizer.cpp:36-43)."""
    return np.concatenate([[256], np.asarray(payload, np.int32), [257]]).astype(np.int32)


def random_text_tokens(seed: int, n: int) -> np.ndarray:
    """SplitMix64 text over a-z + space (proj/tests/acceptance_main.cpp:60-67)."""
    out = np.empty(n, np.int32)
    for i in range(n):
        r = splitmix_at(seed, i) % 27
        out[i] = 32 if r == 26 else 97 + r
    return out


_M64 = (1 << 64) - 1


def splitmix_at(seed: int, i: int) -> int:
    """SplitMix64::at (include/turbokv/rng.hpp:33-38), pure Python."""
    z = (seed + (i + 1) * 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


class Port:
    """The C restatement (oracle/tkv_oracle.c)."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(PORT_SO):
                build(ref=False)
            L = C.CDLL(PORT_SO)
            L.tko_last_error.restype = C.c_char_p
            L.tko_splitmix_at.restype = C.c_uint64
            L.tko_splitmix_at.argtypes = [C.c_uint64, C.c_uint64]
            L.tko_fingerprint_seed.restype = C.c_uint64
            L.tko_chunk_content_id.restype = C.c_uint64
            L.tko_chunk_content_id.argtypes = [C.c_uint64, I32P, C.c_int64]
            L.tko_model_create.argtypes = [C.POINTER(OracleCfg), C.c_uint64, C.POINTER(C.c_void_p)]
            L.tko_model_destroy.argtypes = [C.c_void_p]
            L.tko_weights_checksum.restype = C.c_uint64
            L.tko_weights_checksum.argtypes = [C.c_void_p]
            L.tko_weights_checksum_stream.restype = C.c_uint64
            L.tko_weights_checksum_stream.argtypes = [C.POINTER(OracleCfg), C.c_uint64]
            L.tko_fingerprint_of.restype = C.c_uint64
            L.tko_fingerprint_of.argtypes = [C.POINTER(OracleCfg), C.c_uint64]
            L.tko_model_fingerprint.restype = C.c_uint64
            L.tko_model_fingerprint.argtypes = [C.c_void_p]
            L.tko_weight.restype = F64P
            L.tko_weight.argtypes = [C.c_void_p, C.c_int64, C.c_int, I64P, I64P]
            L.tko_forward.argtypes = [C.c_void_p, I32P, C.c_int64, I64P, F64P, F64P, I64P, C.c_int64,
                                      I64P, I64P, F64P, C.c_int, F64P, F64P]
            L.tko_assemble_positions.argtypes = [I64P, C.c_int64, C.c_int, I64P, I64P]
            L.tko_build_mask_rows.argtypes = [I64P, C.c_int64, C.c_int, I64P, I64P]
            L.tko_causal_rows.argtypes = [C.c_int64, C.c_int64, I64P, I64P]
            L.tko_chunk_kv.argtypes = [C.c_void_p, I32P, C.c_int64, F64P, F64P]
            L.tko_prefill_query.argtypes = [C.c_void_p, F64P, F64P, I64P, C.c_int64, C.c_int64, I32P,
                                            C.c_int64, F64P]
            L.tko_naive_prefill.argtypes = [C.c_void_p, I32P, I64P, C.c_int64, I32P, C.c_int64, C.c_int,
                                            F64P]
            L.tko_rope_rotate.argtypes = [F64P, C.c_int64, C.c_int64, I64P, C.c_int64, C.c_double]
            L.tko_flops_total.restype = C.c_uint64
            L.tko_flops_total.argtypes = [C.POINTER(OracleCfg), C.c_int64, C.c_int64, C.c_int64]
            L.tko_embed.argtypes = [I32P, C.c_int64, C.c_int64, F64P]
            L.tko_top_k.restype = C.c_int64
            L.tko_top_k.argtypes = [F64P, U64P, C.c_int64, C.c_int64, F64P, C.c_int64, U64P, F64P]
            cls._lib = L
        return cls._lib

    def __init__(self, cfg: Cfg, seed: int):
        self.cfg, self.seed = cfg, seed
        L = self.lib()
        h = C.c_void_p()
        self._check(L.tko_model_create(C.byref(cfg.c()), seed, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.lib().tko_model_destroy(self.h)
            self.h = None

    __del__ = close

    def _check(self, rc: int):
        if rc:
            raise OracleError(rc, self.lib().tko_last_error().decode())

    @classmethod
    def stream_identity(cls, cfg: Cfg, seed: int):
        """(checksum, fingerprint) streamed from the generator: no materialised weights (full-size models)."""
        L = cls.lib()
        ck = L.tko_weights_checksum_stream(C.byref(cfg.c()), seed)
        return ck, L.tko_fingerprint_of(C.byref(cfg.c()), ck)

    def checksum(self) -> int:
        return self.lib().tko_weights_checksum(self.h)

    def fingerprint(self) -> int:
        return self.lib().tko_model_fingerprint(self.h)

    def weight(self, layer: int, which: int) -> np.ndarray:
        r, c = C.c_int64(), C.c_int64()
        p = self.lib().tko_weight(self.h, layer, which, C.byref(r), C.byref(c))
        return np.ctypeslib.as_array(p, shape=(r.value, c.value)).copy()

    def chunk_id(self, framed: np.ndarray) -> int:
        framed = np.ascontiguousarray(framed, np.int32)
        return self.lib().tko_chunk_content_id(self.fingerprint(), ptr(framed, I32P), len(framed))

    def chunk_kv(self, framed: np.ndarray):
        framed = np.ascontiguousarray(framed, np.int32)
        L, n, kv = self.cfg.layer_num, len(framed), self.cfg.kv_dim
        k = np.zeros((L, n, kv)); v = np.zeros((L, n, kv))
        self._check(self.lib().tko_chunk_kv(self.h, ptr(framed, I32P), n, ptr(k, F64P), ptr(v, F64P)))
        return k, v

    @staticmethod
    def assemble_positions(lens, reordered: bool):
        lens = np.ascontiguousarray(lens, np.int64)
        pos = np.zeros(int(lens.sum()), np.int64); nxt = C.c_int64()
        Port.lib().tko_assemble_positions(ptr(lens, I64P), len(lens), int(reordered), ptr(pos, I64P),
                                          C.byref(nxt))
        return pos, nxt.value

    def assemble(self, chunks, reordered: bool):
        """Engine::assemble over framed chunks: (K [L,P,kv], V, positions, next_position)."""
        kvs = [self.chunk_kv(c) for c in chunks]
        L, kv = self.cfg.layer_num, self.cfg.kv_dim
        k = np.concatenate([a for a, _ in kvs], axis=1) if kvs else np.zeros((L, 0, kv))
        v = np.concatenate([b for _, b in kvs], axis=1) if kvs else np.zeros((L, 0, kv))
        pos, nxt = self.assemble_positions([len(c) for c in chunks], reordered)
        return np.ascontiguousarray(k), np.ascontiguousarray(v), pos, nxt

    def prefill_query(self, k, v, pos, next_position, q) -> np.ndarray:
        q = np.ascontiguousarray(q, np.int32)
        k = np.ascontiguousarray(k, np.float64); v = np.ascontiguousarray(v, np.float64)
        pos = np.ascontiguousarray(pos, np.int64)
        out = np.zeros(self.cfg.vocab_size)
        self._check(self.lib().tko_prefill_query(self.h, ptr(k, F64P), ptr(v, F64P), ptr(pos, I64P), len(pos),
                                                 next_position, ptr(q, I32P), len(q), ptr(out, F64P)))
        return out

    def naive_prefill(self, chunks, q, independent: bool) -> np.ndarray:
        toks = np.ascontiguousarray(np.concatenate(chunks) if chunks else np.zeros(0), np.int32)
        offs = np.ascontiguousarray(np.concatenate([[0], np.cumsum([len(c) for c in chunks])]), np.int64)
        q = np.ascontiguousarray(q, np.int32)
        out = np.zeros(self.cfg.vocab_size)
        self._check(self.lib().tko_naive_prefill(self.h, ptr(toks, I32P), ptr(offs, I64P), len(chunks),
                                                 ptr(q, I32P), len(q), int(independent), ptr(out, F64P)))
        return out

    def forward(self, tokens, positions, lo, hi, past_k=None, past_v=None, past_pos=None, last_only=False,
                want_kv=False):
        tokens = np.ascontiguousarray(tokens, np.int32)
        positions = np.ascontiguousarray(positions, np.int64)
        lo = np.ascontiguousarray(lo, np.int64); hi = np.ascontiguousarray(hi, np.int64)
        n = len(tokens); L, kv, V = self.cfg.layer_num, self.cfg.kv_dim, self.cfg.vocab_size
        n_past = 0 if past_pos is None else len(past_pos)
        pk = np.ascontiguousarray(past_k if n_past else np.zeros(1), np.float64)
        pv = np.ascontiguousarray(past_v if n_past else np.zeros(1), np.float64)
        pp = np.ascontiguousarray(past_pos if n_past else np.zeros(1), np.int64)
        logits = np.zeros((1 if last_only else n, V))
        nk = np.zeros((L, n, kv)) if want_kv else None
        nv = np.zeros((L, n, kv)) if want_kv else None
        self._check(self.lib().tko_forward(
            self.h, ptr(tokens, I32P), n, ptr(positions, I64P), ptr(pk, F64P), ptr(pv, F64P), ptr(pp, I64P),
            n_past, ptr(lo, I64P), ptr(hi, I64P), ptr(logits, F64P), int(last_only),
            ptr(nk, F64P) if want_kv else None, ptr(nv, F64P) if want_kv else None))
        return (logits, nk, nv) if want_kv else logits

    @staticmethod
    def mask_rows(lens, independent: bool):
        lens = np.ascontiguousarray(lens, np.int64)
        n = int(lens.sum()); lo = np.zeros(n, np.int64); hi = np.zeros(n, np.int64)
        rc = Port.lib().tko_build_mask_rows(ptr(lens, I64P), len(lens), int(independent), ptr(lo, I64P),
                                            ptr(hi, I64P))
        if rc:
            raise OracleError(rc, Port.lib().tko_last_error().decode())
        return lo, hi

    @staticmethod
    def causal_rows(new, past):
        lo = np.zeros(new, np.int64); hi = np.zeros(new, np.int64)
        Port.lib().tko_causal_rows(new, past, ptr(lo, I64P), ptr(hi, I64P))
        return lo, hi

    @staticmethod
    def rope(rows: np.ndarray, positions, head_size: int, base: float = 10000.0) -> np.ndarray:
        out = np.ascontiguousarray(rows, np.float64).copy()
        positions = np.ascontiguousarray(positions, np.int64)
        rc = Port.lib().tko_rope_rotate(ptr(out, F64P), out.shape[0], out.shape[1], ptr(positions, I64P),
                                        head_size, base)
        if rc:
            raise OracleError(rc, Port.lib().tko_last_error().decode())
        return out

    @staticmethod
    def flops_total(cfg: Cfg, n_input, n_context, batch=1) -> int:
        return Port.lib().tko_flops_total(C.byref(cfg.c()), n_input, n_context, batch)

    @staticmethod
    def embed(tokens, dim: int = 256) -> np.ndarray:
        """retrieval.cpp:64-88 restated."""
        t = np.ascontiguousarray(tokens, np.int32)
        out = np.zeros(dim, np.float64)
        rc = Port.lib().tko_embed(ptr(t, I32P), len(t), dim, ptr(out, F64P))
        if rc:
            raise OracleError(rc, Port.lib().tko_last_error().decode())
        return out

    @staticmethod
    def top_k(emb: np.ndarray, ids, query: np.ndarray, k: int):
        """RetrievalIndex::top_k (retrieval.cpp:117-133) restated: (ids, cosines)."""
        emb = np.ascontiguousarray(emb, np.float64)
        idv = np.ascontiguousarray(ids, np.uint64)
        q = np.ascontiguousarray(query, np.float64)
        oi = np.zeros(max(1, min(k, len(idv))), np.uint64)
        os_ = np.zeros(len(oi), np.float64)
        n = Port.lib().tko_top_k(ptr(emb, F64P), ptr(idv, U64P), len(idv), emb.shape[1], ptr(q, F64P), k,
                                 ptr(oi, U64P), ptr(os_, F64P))
        if n < 0:
            raise OracleError(-n, Port.lib().tko_last_error().decode())
        return oi[:n], os_[:n]


class Ref:
    """The reference library itself (proj/src compiled in place + oracle/ref_capi.cpp)."""

    _lib = None

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(REF_SO) or os.path.isdir(REF_SRC)

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(REF_SO):
                build(ref=True)
            L = C.CDLL(REF_SO)
            L.ref_last_error.restype = C.c_char_p
            L.ref_splitmix_at.restype = C.c_uint64
            L.ref_splitmix_at.argtypes = [C.c_uint64, C.c_uint64]
            L.ref_preset.argtypes = [C.c_char_p, C.POINTER(OracleCfg)]
            L.ref_weights_identity.argtypes = [C.POINTER(OracleCfg), C.c_uint64, U64P, U64P, F64P]
            L.ref_weight_tensor.argtypes = [C.POINTER(OracleCfg), C.c_uint64, C.c_int, C.c_int, F64P]
            L.ref_engine_create.argtypes = [C.POINTER(OracleCfg), C.c_uint64, C.c_char_p, C.c_int,
                                            C.POINTER(C.c_void_p)]
            L.ref_engine_destroy.argtypes = [C.c_void_p]
            L.ref_engine_fingerprint.restype = C.c_uint64
            L.ref_engine_fingerprint.argtypes = [C.c_void_p]
            L.ref_ingest.argtypes = [C.c_void_p, I32P, C.c_int64, U64P]
            L.ref_answer.argtypes = [C.c_void_p, C.c_char_p, C.c_int64, C.c_int, C.c_int64, U64P, C.c_int64, I64P,
                                     I32P, C.c_int64, I64P, U64P]
            L.ref_chunk_document.argtypes = [C.c_char_p, C.c_int64, C.c_int64, I64P, C.c_int64, I64P]
            L.ref_bench_ingest.argtypes = [C.c_void_p, I64P, C.c_int64, C.c_uint64, U64P, C.c_int64, I64P]
            L.ref_store_path.argtypes = [C.c_void_p, C.c_uint64, C.c_char_p, C.c_int64]
            L.ref_assemble.argtypes = [C.c_void_p, U64P, C.c_int64, C.c_int, C.POINTER(C.c_void_p)]
            L.ref_ctx_destroy.argtypes = [C.c_void_p]
            L.ref_ctx_total_tokens.restype = C.c_int64
            L.ref_ctx_total_tokens.argtypes = [C.c_void_p]
            L.ref_ctx_info.argtypes = [C.c_void_p, I64P, I64P]
            L.ref_ctx_kv.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, F64P]
            L.ref_prefill_query.argtypes = [C.c_void_p, C.c_void_p, I32P, C.c_int64, F64P, U64P]
            L.ref_naive_prefill.argtypes = [C.c_void_p, I32P, I64P, C.c_int64, I32P, C.c_int64, C.c_int, F64P,
                                            C.POINTER(C.c_void_p)]
            L.ref_greedy_decode.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, I32P, I64P]
            L.ref_set_inject_fault.argtypes = [C.c_int]
            L.ref_save_weights.argtypes = [C.POINTER(OracleCfg), C.c_uint64, C.c_char_p]
            L.ref_load_weights.argtypes = [C.c_char_p, C.POINTER(OracleCfg), U64P]
            L.ref_forward_file.argtypes = [C.c_char_p, I32P, C.c_int64, F64P]
            L.ref_build_mask.argtypes = [I64P, C.c_int64, C.c_int, U8P]
            L.ref_causal_rows.argtypes = [C.c_int64, C.c_int64, U8P]
            L.ref_rope_rotate.argtypes = [F64P, C.c_int64, C.c_int64, I64P, C.c_int64, C.c_double, F64P]
            L.ref_attend.argtypes = [F64P, C.c_int64, F64P, F64P, C.c_int64, C.c_int64, C.c_int64, U8P,
                                     C.c_int64, F64P]
            L.ref_flops_compare.argtypes = [C.POINTER(OracleCfg), C.c_int64, C.c_int64, C.c_int64, U64P, U64P,
                                            F64P]
            L.ref_embed.argtypes = [I32P, C.c_int64, C.c_int64, F64P]
            L.ref_top_k.argtypes = [F64P, U64P, C.c_int64, C.c_int64, F64P, C.c_int64, U64P, I64P]
            cls._lib = L
        return cls._lib

    @classmethod
    def check(cls, rc: int):
        if rc:
            raise OracleError(rc, cls.lib().ref_last_error().decode())

    @classmethod
    def embed(cls, tokens, dim: int = 256) -> np.ndarray:
        t = np.ascontiguousarray(tokens, np.int32)
        out = np.zeros(dim, np.float64)
        cls.check(cls.lib().ref_embed(ptr(t, I32P), len(t), dim, ptr(out, F64P)))
        return out

    @classmethod
    def top_k(cls, emb: np.ndarray, ids, query: np.ndarray, k: int) -> np.ndarray:
        emb = np.ascontiguousarray(emb, np.float64)
        idv = np.ascontiguousarray(ids, np.uint64)
        q = np.ascontiguousarray(query, np.float64)
        out = np.zeros(max(1, min(k, len(idv))), np.uint64)
        n = C.c_int64()
        cls.check(cls.lib().ref_top_k(ptr(emb, F64P), ptr(idv, U64P), len(idv), emb.shape[1], ptr(q, F64P), k,
                                      ptr(out, U64P), C.byref(n)))
        return out[:n.value]

    @classmethod
    def identity(cls, cfg: Cfg, seed: int):
        ck, fp, e = C.c_uint64(), C.c_uint64(), C.c_double()
        cls.check(cls.lib().ref_weights_identity(C.byref(cfg.c()), seed, C.byref(ck), C.byref(fp), C.byref(e)))
        return ck.value, fp.value, e.value

    @classmethod
    def build_mask(cls, lens, independent: bool) -> np.ndarray:
        lens = np.ascontiguousarray(lens, np.int64); n = int(lens.sum())
        out = np.zeros((n, n), np.uint8)
        cls.check(cls.lib().ref_build_mask(ptr(lens, I64P), len(lens), int(independent), ptr(out, U8P)))
        return out

    @classmethod
    def causal_rows(cls, new, past) -> np.ndarray:
        out = np.zeros((new, past + new), np.uint8)
        cls.check(cls.lib().ref_causal_rows(new, past, ptr(out, U8P)))
        return out


def ref_chunk_lengths(text: bytes, target_len: int) -> list:
    """The reference's chunk_document (retrieval.cpp:32-58): byte length of every chunk, in order."""
    out = np.zeros(max(1, len(text)), np.int64)
    n = C.c_int64()
    Ref.check(Ref.lib().ref_chunk_document(text, len(text), target_len, ptr(out, I64P), len(out), C.byref(n)))
    return [int(x) for x in out[:n.value]]


class RefEngine:
    """turbokv::Engine driven through oracle/ref_capi.cpp (TKVC store on disk)."""

    def __init__(self, cfg: Cfg, seed: int, store_root: str, f32_store: bool = False):
        self.cfg = cfg
        L = Ref.lib()
        h = C.c_void_p()
        Ref.check(L.ref_engine_create(C.byref(cfg.c()), seed, store_root.encode(), 2 if f32_store else 1,
                                      C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            Ref.lib().ref_engine_destroy(self.h)
            self.h = None

    __del__ = close

    def fingerprint(self) -> int:
        return Ref.lib().ref_engine_fingerprint(self.h)

    def ingest(self, payload) -> int:
        payload = np.ascontiguousarray(payload, np.int32)
        out = C.c_uint64()
        Ref.check(Ref.lib().ref_ingest(self.h, ptr(payload, I32P), len(payload), C.byref(out)))
        return out.value

    def answer(self, question: str, k: int, mode: int, max_new: int) -> dict:
        """Engine::answer: retrieved ids, tokens, counters."""
        ids = np.zeros(256, np.uint64)
        toks = np.zeros(max(max_new, 1), np.int32)
        st = np.zeros(5, np.uint64)
        ni, nt = C.c_int64(), C.c_int64()
        Ref.check(Ref.lib().ref_answer(self.h, question.encode(), k, mode, max_new, ptr(ids, U64P), len(ids),
                                       C.byref(ni), ptr(toks, I32P), len(toks), C.byref(nt), ptr(st, U64P)))
        return {"retrieved": [int(x) for x in ids[:ni.value]], "tokens": [int(x) for x in toks[:nt.value]],
                "prefill_flops": int(st[0]), "modeled_prefill_flops": int(st[1]), "decode_flops": int(st[2]),
                "context_tokens": int(st[3]), "query_tokens": int(st[4])}

    def bench_ingest(self, doc_grid, seed: int) -> list:
        """bench.cpp ingest_synthetic: the reference's bench corpus, chunk ids in ingest order."""
        grid = np.ascontiguousarray(doc_grid, np.int64)
        out = np.zeros(4096, np.uint64)
        n = C.c_int64()
        Ref.check(Ref.lib().ref_bench_ingest(self.h, ptr(grid, I64P), len(grid), seed, ptr(out, U64P), len(out),
                                             C.byref(n)))
        return [int(x) for x in out[:n.value]]

    def store_path(self, chunk_id: int) -> str:
        buf = C.create_string_buffer(4096)
        Ref.check(Ref.lib().ref_store_path(self.h, chunk_id, buf, 4096))
        return buf.value.decode()

    def assemble(self, ids, reordered: bool) -> "RefCtx":
        ids = np.ascontiguousarray(ids, np.uint64)
        h = C.c_void_p()
        Ref.check(Ref.lib().ref_assemble(self.h, ptr(ids, U64P), len(ids), int(reordered), C.byref(h)))
        return RefCtx(self, h)

    def naive_prefill(self, chunks, q, independent: bool, keep_ctx=False):
        toks = np.ascontiguousarray(np.concatenate(chunks) if chunks else np.zeros(0), np.int32)
        offs = np.ascontiguousarray(np.concatenate([[0], np.cumsum([len(c) for c in chunks])]), np.int64)
        q = np.ascontiguousarray(q, np.int32)
        out = np.zeros(self.cfg.vocab_size)
        h = C.c_void_p()
        Ref.check(Ref.lib().ref_naive_prefill(self.h, ptr(toks, I32P), ptr(offs, I64P), len(chunks),
                                              ptr(q, I32P), len(q), int(independent), ptr(out, F64P),
                                              C.byref(h) if keep_ctx else None))
        return (out, RefCtx(self, h)) if keep_ctx else out


class RefCtx:
    def __init__(self, eng: RefEngine, h):
        self.eng, self.h = eng, h

    def close(self):
        if getattr(self, "h", None):
            Ref.lib().ref_ctx_destroy(self.h)
            self.h = None

    __del__ = close

    def total_tokens(self) -> int:
        return Ref.lib().ref_ctx_total_tokens(self.h)

    def positions(self):
        n = self.total_tokens()
        pos = np.zeros(max(n, 1), np.int64); nxt = C.c_int64()
        Ref.check(Ref.lib().ref_ctx_info(self.h, ptr(pos, I64P), C.byref(nxt)))
        return pos[:n], nxt.value

    def kv(self, layer: int, which: int) -> np.ndarray:
        """which: 0 K unrotated, 1 V, 2 K rotated by the context's positions."""
        out = np.zeros((self.total_tokens(), self.eng.cfg.kv_dim))
        Ref.check(Ref.lib().ref_ctx_kv(self.eng.h, self.h, layer, which, ptr(out, F64P)))
        return out

    def prefill_query(self, q):
        q = np.ascontiguousarray(q, np.int32)
        out = np.zeros(self.eng.cfg.vocab_size); fl = np.zeros(4, np.uint64)
        Ref.check(Ref.lib().ref_prefill_query(self.eng.h, self.h, ptr(q, I32P), len(q), ptr(out, F64P),
                                              ptr(fl, U64P)))
        return out, fl

    def greedy_decode(self, max_new: int) -> np.ndarray:
        out = np.zeros(max(max_new, 1), np.int32); n = C.c_int64()
        Ref.check(Ref.lib().ref_greedy_decode(self.eng.h, self.h, max_new, ptr(out, I32P), C.byref(n)))
        return out[:n.value]
