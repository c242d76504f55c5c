"""Python mirror of the reference `turbokv` C++ API over the C ABI (include/tkv.h).

Names, argument meaning and error classes follow /root/reference/proj/include/turbokv/*.hpp
so parity tests read like the reference's own tests:

    Engine(config, seed)                    pipeline.hpp:69-72
    Engine.ingest_chunk_payload(doc, toks)  pipeline.hpp:86-88
    Engine.assemble(ids, PositionMode)      pipeline.hpp:93
    Engine.prefill_query(ctx, toks)         pipeline.hpp:97-99
    Engine.naive_prefill(chunks, q, mode)   pipeline.hpp:104-108
    greedy_decode(...)                      model.hpp:74-81
    errors                                   errors.hpp:10-67

Every call goes through libtkv_b200.so (sm_100a kernels). There is no CPU fallback: without the
built library or a B200 the import / Engine() raises.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TKV_LIB_PATH") or os.path.join(_HERE, "libtkv_b200.so")  # override: variant builds (tools/)

I32P, I64P, U64P = C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_uint64)
F32P, U8P = C.POINTER(C.c_float), C.POINTER(C.c_uint8)


class Error(RuntimeError):
    """turbokv::Error"""


class ShapeError(Error): pass
class DomainError(Error): pass
class ConfigError(Error): pass
class DegenerateRowError(Error): pass
class IoError(Error): pass
class FormatError(Error): pass
class NotFoundError(Error): pass
class StaleCacheError(Error): pass
class NoContextError(Error): pass
class CudaError(Error): pass
class OutOfMemoryError(Error): pass


_ERRORS = {1: Error, 2: ShapeError, 3: DomainError, 4: ConfigError, 5: DegenerateRowError, 6: IoError,
           7: FormatError, 8: NotFoundError, 9: StaleCacheError, 10: NoContextError, 11: CudaError,
           12: OutOfMemoryError}


class PositionMode(enum.IntEnum):
    Composite = 0
    Reordered = 1


class MaskMode(enum.IntEnum):
    Causal = 0
    Independent = 1


class Dtype(enum.IntEnum):
    F32 = 1
    BF16 = 2


FLAG_SIMT_GEMM = 0x1
FLAG_SIMT_ATTN = 0x2
FLAG_NO_PDL = 0x8
FLAG_NO_GRAPHS = 0x100
FLAG_BATCH_ATTN = 0x20
FLAG_DECODE_ATTN = 0x40

DOC_START, DOC_END, EOS, VOCAB = 256, 257, 258, 259  # tokenizer.hpp:19-22


class _Cfg(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("layer_num", "head_num", "kv_head_num", "head_size", "hidden_size",
                                          "intermediate_size", "vocab_size")] + \
               [("rope_base", C.c_double), ("norm_eps", C.c_double)]


class _Opts(C.Structure):
    _fields_ = [("dtype", C.c_int), ("device", C.c_int32), ("page_tokens", C.c_int32),
                ("store_capacity_tokens", C.c_int64), ("max_position", C.c_int64),
                ("exact_fingerprint", C.c_int32), ("flags", C.c_int32), ("host_spill_tokens", C.c_int64)]


class _Stats(C.Structure):
    _fields_ = [("chunks", C.c_int64), ("new_chunks", C.c_int64), ("bytes_written", C.c_uint64)]


class _Ipc(C.Structure):
    _fields_ = [("bytes", C.c_uint8 * 64)]


class _Flops(C.Structure):
    _fields_ = [("qkv", C.c_uint64), ("attn", C.c_uint64), ("o", C.c_uint64), ("mlp", C.c_uint64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built: run `make -C {_HERE}` (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        L.tkv_last_error.restype = C.c_char_p
        L.tkv_status_name.restype = C.c_char_p
        L.tkv_config_preset.argtypes = [C.c_char_p, C.POINTER(_Cfg)]
        L.tkv_config_validate.argtypes = [C.POINTER(_Cfg)]
        L.tkv_config_fingerprint_seed.restype = C.c_uint64
        L.tkv_config_fingerprint_seed.argtypes = [C.POINTER(_Cfg)]
        L.tkv_weights_identity.argtypes = [C.POINTER(_Cfg), C.c_uint64, U64P, U64P]
        L.tkv_kernel_timeline.argtypes = [C.c_void_p, C.c_int, U64P, I32P, C.c_int64, C.POINTER(C.c_int64)]
        L.tkv_debug_weights_checksum.argtypes = [C.POINTER(_Cfg), C.c_uint64, C.c_int, U64P, U64P]
        L.tkv_engine_check.argtypes = [C.c_void_p]
        L.tkv_debug_weight_rows.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int64, C.c_int64, F32P]
        L.tkv_chunk_content_id.restype = C.c_uint64
        L.tkv_chunk_content_id.argtypes = [C.c_uint64, I32P, C.c_int64]
        L.tkv_engine_opts_default.argtypes = [C.POINTER(_Opts)]
        L.tkv_engine_create.argtypes = [C.POINTER(_Cfg), C.c_uint64, C.POINTER(_Opts), C.POINTER(C.c_void_p)]
        L.tkv_engine_destroy.argtypes = [C.c_void_p]
        L.tkv_engine_create_from_weights.argtypes = [C.c_char_p, C.POINTER(_Opts), C.POINTER(C.c_void_p), C.POINTER(_Cfg)]
        L.tkv_save_weights.argtypes = [C.POINTER(_Cfg), C.c_uint64, C.c_char_p, C.c_int]
        L.tkv_engine_fingerprint.argtypes = [C.c_void_p, U64P]
        L.tkv_ingest_chunks.argtypes = [C.c_void_p, I32P, I64P, C.c_int64, U64P, C.POINTER(_Stats)]
        L.tkv_import_tkvc.argtypes = [C.c_void_p, C.c_char_p, U64P]
        L.tkv_export_tkvc.argtypes = [C.c_void_p, C.c_uint64, C.c_char_p]
        L.tkv_store_contains.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_int)]
        L.tkv_store_chunk_tokens.argtypes = [C.c_void_p, C.c_uint64, I64P]
        L.tkv_store_count.argtypes = [C.c_void_p, I64P, I64P, I64P]
        L.tkv_store_ids.argtypes = [C.c_void_p, U64P, C.c_int64, I64P]
        L.tkv_store_evict.argtypes = [C.c_void_p, C.c_uint64]
        L.tkv_embed.argtypes = [I32P, C.c_int64, C.c_int64, C.POINTER(C.c_double)]
        L.tkv_index_add.argtypes = [C.c_void_p, C.c_uint64, I32P, C.c_int64, C.POINTER(C.c_int)]
        L.tkv_index_size.restype = C.c_int64
        L.tkv_index_size.argtypes = [C.c_void_p]
        L.tkv_index_top_k.argtypes = [C.c_void_p, I32P, C.c_int64, C.c_int64, U64P, C.POINTER(C.c_double), I64P]
        L.tkv_store_tiers.argtypes = [C.c_void_p, I64P, I64P, I64P, I64P]
        L.tkv_store_chunk_tier.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_int32)]
        L.tkv_prefill_query_batch.argtypes = [C.c_void_p, C.POINTER(C.c_void_p), C.c_int64, I32P, I64P, F32P,
                                              C.POINTER(_Flops)]
        L.tkv_store_read.argtypes = [C.c_void_p, C.c_uint64, C.c_int64, C.c_int, F32P, C.c_int64]
        L.tkv_assemble.argtypes = [C.c_void_p, U64P, C.c_int64, C.c_int, C.POINTER(C.c_void_p)]
        L.tkv_prefill_query.argtypes = [C.c_void_p, C.c_void_p, I32P, C.c_int64, F32P, C.POINTER(_Flops)]
        L.tkv_prefill_query_device.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
        L.tkv_naive_prefill.argtypes = [C.c_void_p, I32P, I64P, C.c_int64, I32P, C.c_int64, C.c_int, F32P,
                                        C.POINTER(_Flops), C.POINTER(C.c_void_p)]
        L.tkv_naive_prefill_ids.argtypes = [C.c_void_p, U64P, C.c_int64, I32P, C.c_int64, C.c_int, F32P,
                                            C.POINTER(_Flops), C.POINTER(C.c_void_p)]
        L.tkv_greedy_decode.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, I32P, I64P]
        L.tkv_context_destroy.argtypes = [C.c_void_p]
        L.tkv_context_total_tokens.restype = C.c_int64
        L.tkv_context_total_tokens.argtypes = [C.c_void_p]
        L.tkv_context_next_position.restype = C.c_int64
        L.tkv_context_next_position.argtypes = [C.c_void_p]
        L.tkv_context_segments.restype = C.c_int64
        L.tkv_context_segments.argtypes = [C.c_void_p, I64P, I32P, C.c_int64]
        L.tkv_context_positions.argtypes = [C.c_void_p, I64P, C.c_int64]
        L.tkv_context_last_logits.argtypes = [C.c_void_p, F32P, C.c_int64]
        L.tkv_context_read_kv.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, F32P, C.c_int64]
        L.tkv_context_mask.argtypes = [C.c_void_p, U8P, C.c_int64, C.c_int64]
        L.tkv_engine_stream.restype = C.c_void_p
        L.tkv_engine_stream.argtypes = [C.c_void_p]
        L.tkv_profile_enable.argtypes = [C.c_void_p, C.c_int]
        L.tkv_profile_read.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_double), I64P]
        L.tkv_profile_reset.argtypes = [C.c_void_p]
        L.tkv_io_bytes.argtypes = [C.c_void_p, I64P, I64P]
        L.tkv_launch_count.restype = C.c_int64
        L.tkv_launch_count.argtypes = [C.c_void_p]
        L.tkv_debug_set_mask_fault.argtypes = [C.c_void_p, C.c_int64, C.c_int64]
        L.tkv_debug_set_mask_rows.argtypes = [C.c_void_p, I64P, I32P, I32P, C.c_int64]
        L.tkv_store_export_ipc.argtypes = [C.c_void_p, C.POINTER(_Ipc), C.POINTER(C.c_uint64)]
        L.tkv_store_attach_ipc.argtypes = [C.c_void_p, C.c_int32, C.POINTER(_Ipc)]
        L.tkv_store_attach_engine.argtypes = [C.c_void_p, C.c_int32, C.c_void_p]
        L.tkv_store_chunk_pages.argtypes = [C.c_void_p, C.c_uint64, I32P, C.c_int64, I64P, I64P]
        L.tkv_store_register_remote.argtypes = [C.c_void_p, C.c_uint64, C.c_int32, C.c_int64, I32P, C.c_int64, I32P]
        L.tkv_store_fetch_remote.argtypes = [C.c_void_p, C.c_uint64]
        L.tkv_store_rebalance.argtypes = [C.c_void_p, C.c_int64, I64P, I64P]
        L.tkv_store_export_directory.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, I64P]
        L.tkv_store_import_directory.argtypes = [C.c_void_p, C.c_int32, C.c_char_p, C.c_int64]
        L.tkv_remote_bytes.restype = C.c_int64
        L.tkv_remote_bytes.argtypes = [C.c_void_p]
        L.tkv_debug_attn_trace.argtypes = [C.c_int, U64P, C.c_int64]
        L.tkv_debug_set_gemm_knobs.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int]
        L.tkv_debug_gemm_trace.argtypes = [C.c_int, U64P, C.c_int64]
        L.tkv_debug_gemm_bench.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int,
                                           C.POINTER(C.c_double)]
        L.tkv_debug_gemm.argtypes = [C.c_int, C.c_int, C.c_int, F32P, F32P, C.c_int64, C.c_int64, C.c_int64,
                                     C.c_int, F32P]
        L.tkv_debug_attention.argtypes = [C.c_int, C.c_int, C.c_int, F32P, F32P, F32P, I32P, I32P, C.c_int64,
                                          C.c_int64, C.c_int64, C.c_int64, C.c_int64, F32P]
        _lib = L
    return _lib


def _check(rc: int):
    if rc:
        raise _ERRORS.get(rc, Error)(lib().tkv_last_error().decode(errors="replace"))


def _p(a, t):
    return a.ctypes.data_as(t)


def _i32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.int32))


@dataclass
class ModelConfig:
    """include/turbokv/config.hpp:11-34"""
    layer_num: int = 0
    head_num: int = 0
    kv_head_num: int = 0
    head_size: int = 0
    hidden_size: int = 0
    intermediate_size: int = 0
    vocab_size: int = 0
    rope_base: float = 10000.0
    norm_eps: float = 1e-6

    def _c(self) -> _Cfg:
        return _Cfg(self.layer_num, self.head_num, self.kv_head_num, self.head_size, self.hidden_size,
                    self.intermediate_size, self.vocab_size, self.rope_base, self.norm_eps)

    @staticmethod
    def preset(name: str) -> "ModelConfig":
        c = _Cfg()
        _check(lib().tkv_config_preset(name.encode(), C.byref(c)))
        return ModelConfig(*(getattr(c, f[0]) for f in _Cfg._fields_))

    @staticmethod
    def toy() -> "ModelConfig":
        return ModelConfig.preset("toy")

    @staticmethod
    def qwen2_7b_like() -> "ModelConfig":
        return ModelConfig.preset("qwen2-7b")

    @staticmethod
    def llama3_8b_like() -> "ModelConfig":
        return ModelConfig.preset("llama3-8b")

    def validate(self) -> None:
        _check(lib().tkv_config_validate(C.byref(self._c())))

    def fingerprint_seed(self) -> int:
        return lib().tkv_config_fingerprint_seed(C.byref(self._c()))

    @property
    def kv_dim(self) -> int:
        return self.kv_head_num * self.head_size


@dataclass
class IngestStats:
    chunks: int = 0
    new_chunks: int = 0
    bytes_written: int = 0


@dataclass
class FlopCounter:
    """costmodel.hpp:53-63"""
    qkv: int = 0
    attn: int = 0
    o: int = 0
    mlp: int = 0

    def total(self) -> int:
        return self.qkv + self.attn + self.o + self.mlp

    def _add(self, f: _Flops):
        self.qkv += f.qkv
        self.attn += f.attn
        self.o += f.o
        self.mlp += f.mlp


def weights_identity(config: ModelConfig, seed: int):
    """(weights_checksum, model_fingerprint) — model.cpp:94-118."""
    ck, fp = C.c_uint64(), C.c_uint64()
    _check(lib().tkv_weights_identity(C.byref(config._c()), seed, C.byref(ck), C.byref(fp)))
    return ck.value, fp.value


def save_weights(config: ModelConfig, seed: int, path: str, device: int = 0) -> None:
    """TKVW file of init_random(config, seed) (tkv_save_weights; byte-identical to the reference's save_weights)."""
    _check(lib().tkv_save_weights(C.byref(config._c()), seed, str(path).encode(), device))


def weights_identity_device(config: ModelConfig, seed: int, device: int = 0):
    """(weights_checksum, model_fingerprint) hashed on GPU `device` (the engine's path, fingerprint.cu)."""
    ck, fp = C.c_uint64(), C.c_uint64()
    _check(lib().tkv_debug_weights_checksum(C.byref(config._c()), seed, device, C.byref(ck), C.byref(fp)))
    return ck.value, fp.value


def chunk_content_id(framed, model_fingerprint: int) -> int:
    """kvstore.cpp:58-64"""
    f = _i32(framed)
    return lib().tkv_chunk_content_id(model_fingerprint, _p(f, I32P), len(f))


def frame_chunk(payload) -> np.ndarray:
    """tok::frame_chunk (tokenizer.cpp:36-43)"""
    return np.concatenate([[DOC_START], np.asarray(payload, np.int32), [DOC_END]]).astype(np.int32)


def encode(text: str) -> np.ndarray:
    """tok::encode (tokenizer.cpp:8-15)"""
    return np.frombuffer(text.encode(), dtype=np.uint8).astype(np.int32)


class AssembledContext:
    """include/turbokv/context.hpp:16-38 — handle on a request cache in HBM."""

    def __init__(self, engine: "Engine", handle):
        self.engine, self._h = engine, handle

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            lib().tkv_context_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def total_tokens(self) -> int:
        return lib().tkv_context_total_tokens(self._h)

    @property
    def next_position(self) -> int:
        return lib().tkv_context_next_position(self._h)

    @property
    def positions(self) -> np.ndarray:
        n = self.total_tokens()
        out = np.zeros(max(n, 1), np.int64)
        _check(lib().tkv_context_positions(self._h, _p(out, I64P), len(out)))
        return out[:n]

    @property
    def segments(self):
        n = lib().tkv_context_segments(self._h, None, None, 0)
        lens = np.zeros(max(n, 1), np.int64)
        q = np.zeros(max(n, 1), np.int32)
        lib().tkv_context_segments(self._h, _p(lens, I64P), _p(q, I32P), n)
        return [(int(lens[i]), "query" if q[i] else "chunk") for i in range(n)]

    @property
    def last_logits(self) -> np.ndarray:
        out = np.zeros(self.engine.config.vocab_size, np.float32)
        _check(lib().tkv_context_last_logits(self._h, _p(out, F32P), len(out)))
        return out[None, :]

    def prefilled(self) -> bool:
        try:
            self.last_logits
            return True
        except DomainError:
            return False

    def read_kv(self, layer: int, which: str = "k", rotated: bool = False) -> np.ndarray:
        n = self.total_tokens()
        out = np.zeros((n, self.engine.config.kv_dim), np.float32)
        _check(lib().tkv_context_read_kv(self._h, layer, 0 if which == "k" else 1, int(rotated),
                                         _p(out, F32P), out.size))
        return out

    def mask(self, rows: int, cols: int) -> np.ndarray:
        out = np.zeros((rows, cols), np.uint8)
        _check(lib().tkv_context_mask(self._h, _p(out, U8P), rows, cols))
        return out


class Engine:
    """turbokv::Engine (include/turbokv/pipeline.hpp:64-131) on one B200."""

    def __init__(self, config: ModelConfig, seed: int, dtype: str | Dtype = "bf16", device: int = 0,
                 page_tokens: int = 64, store_capacity_tokens: int = 0, max_position: int = 0,
                 exact_fingerprint: int = -1, flags: int = 0, host_spill_tokens: int = 0, weights_path: str | None = None):
        """Weights from (config, seed) in init_random's draw order, or -- weights_path -- from a TKVW file (the config
        is then read from the file; `config` may be None)."""
        self.config = config
        self.seed = seed
        self._framed = {}  # chunk id -> framed tokens (host copy for the naive path / answer)
        o = _Opts()
        lib().tkv_engine_opts_default(C.byref(o))
        o.dtype = int(Dtype.F32 if str(dtype).lower() in ("f32", "fp32", "float32", "dtype.f32") or dtype == Dtype.F32
                      else Dtype.BF16)
        o.device, o.page_tokens, o.store_capacity_tokens = device, page_tokens, store_capacity_tokens
        o.max_position, o.exact_fingerprint, o.flags = max_position, exact_fingerprint, flags
        o.host_spill_tokens = host_spill_tokens
        self.dtype = Dtype(o.dtype)
        h = C.c_void_p()
        if weights_path is not None:
            c = _Cfg()
            _check(lib().tkv_engine_create_from_weights(str(weights_path).encode(), C.byref(o), C.byref(h), C.byref(c)))
            self.config = ModelConfig(*[getattr(c, f) for f, _ in _Cfg._fields_])
        else:
            _check(lib().tkv_engine_create(C.byref(config._c()), seed, C.byref(o), C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().tkv_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def fingerprint(self) -> int:
        out = C.c_uint64()
        _check(lib().tkv_engine_fingerprint(self._h, C.byref(out)))
        return out.value

    def check(self) -> None:
        """Synchronise the engine stream and raise deferred device errors (tkv_engine_check)."""
        _check(lib().tkv_engine_check(self._h))

    def weight_rows(self, layer: int, which: int, row0: int, nrows: int, cols: int) -> np.ndarray:
        """Device weight rows as float32 (tkv_debug_weight_rows; layout in include/tkv.h)."""
        out = np.zeros((nrows, cols), np.float32)
        _check(lib().tkv_debug_weight_rows(self._h, layer, which, row0, nrows, _p(out, F32P)))
        return out

    # ---- offline precompute ----
    def ingest_chunks(self, payloads, stats: IngestStats | None = None) -> list[int]:
        payloads = [np.asarray(p, np.int32) for p in payloads]
        flat = _i32(np.concatenate(payloads) if payloads else np.zeros(0))
        offs = np.ascontiguousarray(np.concatenate([[0], np.cumsum([len(p) for p in payloads])]), np.int64)
        ids = np.zeros(max(len(payloads), 1), np.uint64)
        st = _Stats()
        _check(lib().tkv_ingest_chunks(self._h, _p(flat, I32P), _p(offs, I64P), len(payloads), _p(ids, U64P),
                                       C.byref(st)))
        if stats is not None:
            stats.chunks += st.chunks
            stats.new_chunks += st.new_chunks
            stats.bytes_written += st.bytes_written
        out = [int(i) for i in ids[:len(payloads)]]
        for cid, p in zip(out, payloads):
            self._framed.setdefault(cid, np.concatenate([[256], p, [257]]).astype(np.int32))
        return out

    def ingest_chunk_payload(self, doc_id: str, payload, stats: IngestStats | None = None) -> int:
        return self.ingest_chunks([payload], stats)[0]

    def import_tkvc(self, path: str) -> int:
        out = C.c_uint64()
        _check(lib().tkv_import_tkvc(self._h, path.encode(), C.byref(out)))
        return out.value

    def export_tkvc(self, chunk_id: int, path: str) -> None:
        _check(lib().tkv_export_tkvc(self._h, chunk_id, path.encode()))

    # ---- retrieval (retrieval.hpp) ----
    def index_add(self, chunk_id: int, payload) -> bool:
        p = _i32(payload)
        a = C.c_int()
        _check(lib().tkv_index_add(self._h, chunk_id, _p(p, I32P) if len(p) else None, len(p), C.byref(a)))
        return bool(a.value)

    def index_size(self) -> int:
        return lib().tkv_index_size(self._h)

    def top_k(self, query_tokens, k: int):
        """RetrievalIndex::top_k over embed(query): (chunk ids, cosines), best first."""
        q = _i32(query_tokens)
        n = max(1, min(int(k), max(1, self.index_size()), 256))
        ids = np.zeros(n, np.uint64)
        sc = np.zeros(n, np.float64)
        got = C.c_int64()
        _check(lib().tkv_index_top_k(self._h, _p(q, I32P) if len(q) else None, len(q), k, _p(ids, U64P),
                                     sc.ctypes.data_as(C.POINTER(C.c_double)), C.byref(got)))
        return ids[:got.value], sc[:got.value]

    def store_tiers(self) -> dict:
        v = [C.c_int64() for _ in range(4)]
        _check(lib().tkv_store_tiers(self._h, *[C.byref(x) for x in v]))
        return {"hbm_used": v[0].value, "hbm_total": v[1].value, "host_used": v[2].value, "host_total": v[3].value}

    def store_chunk_tier(self, chunk_id: int) -> int:
        """0 = HBM, 1 = pinned host spill tier, 2 = a peer GPU's pool."""
        t = C.c_int32()
        _check(lib().tkv_store_chunk_tier(self._h, chunk_id, C.byref(t)))
        return t.value

    def store_evict(self, chunk_id: int) -> None:
        _check(lib().tkv_store_evict(self._h, chunk_id))
        self._framed.pop(chunk_id, None)

    def store_contains(self, chunk_id: int) -> bool:
        out = C.c_int()
        _check(lib().tkv_store_contains(self._h, chunk_id, C.byref(out)))
        return bool(out.value)

    def store_chunk_tokens(self, chunk_id: int) -> int:
        n = C.c_int64()
        _check(lib().tkv_store_chunk_tokens(self._h, chunk_id, C.byref(n)))
        return n.value

    def chunk_framed_tokens(self, chunk_id: int) -> np.ndarray:
        """The framed tokens a chunk was ingested from (ChunkRecord::tokens, retrieval.hpp:25-30): kept host-side
        for the full-concat comparison path."""
        if chunk_id not in self._framed:
            raise NotFoundError(f"chunk {chunk_id:016x}: tokens not held by this engine")
        return self._framed[chunk_id]

    def store_ids(self) -> list:
        """CacheStore::ids: every stored chunk id, ascending."""
        n = C.c_int64()
        _check(lib().tkv_store_ids(self._h, None, 0, C.byref(n)))
        out = np.zeros(max(n.value, 1), np.uint64)
        _check(lib().tkv_store_ids(self._h, _p(out, U64P), len(out), C.byref(n)))
        return [int(x) for x in out[:n.value]]

    def store_read(self, chunk_id: int, layer: int, which: str = "k") -> np.ndarray:
        n = C.c_int64()
        _check(lib().tkv_store_chunk_tokens(self._h, chunk_id, C.byref(n)))
        out = np.zeros((n.value, self.config.kv_dim), np.float32)
        _check(lib().tkv_store_read(self._h, chunk_id, layer, 0 if which == "k" else 1, _p(out, F32P), out.size))
        return out

    def store_count(self):
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        _check(lib().tkv_store_count(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    # ---- online path ----
    def assemble(self, chunk_ids, mode: PositionMode = PositionMode.Reordered) -> AssembledContext:
        ids = np.ascontiguousarray(np.asarray(list(chunk_ids), dtype=np.uint64))
        h = C.c_void_p()
        _check(lib().tkv_assemble(self._h, _p(ids, U64P) if len(ids) else None, len(ids), int(mode), C.byref(h)))
        return AssembledContext(self, h)

    def prefill_query(self, ctx: AssembledContext, query_tokens, counter: FlopCounter | None = None) -> np.ndarray:
        q = _i32(query_tokens)
        out = np.zeros(self.config.vocab_size, np.float32)
        fl = _Flops()
        _check(lib().tkv_prefill_query(self._h, ctx.handle, _p(q, I32P) if len(q) else None, len(q),
                                       _p(out, F32P), C.byref(fl)))
        if counter is not None:
            counter._add(fl)
        return out[None, :]

    def prefill_query_batch(self, ctxs, queries, counter: FlopCounter | None = None) -> np.ndarray:
        """tkv_prefill_query_batch: one forward over every request's query tokens; returns [n_req, vocab]."""
        qs = [_i32(q) for q in queries]
        flat = _i32(np.concatenate(qs))
        offs = np.ascontiguousarray(np.concatenate([[0], np.cumsum([len(q) for q in qs])]), np.int64)
        hs = (C.c_void_p * len(ctxs))(*[c.handle for c in ctxs])
        out = np.zeros((len(ctxs), self.config.vocab_size), np.float32)
        fl = _Flops()
        _check(lib().tkv_prefill_query_batch(self._h, hs, len(ctxs), _p(flat, I32P), _p(offs, I64P), _p(out, F32P),
                                             C.byref(fl)))
        if counter is not None:
            counter._add(fl)
        return out

    def prefill_query_device(self, ctx: AssembledContext, d_tokens: int, n: int, d_logits: int) -> None:
        _check(lib().tkv_prefill_query_device(self._h, ctx.handle, C.c_void_p(d_tokens), n, C.c_void_p(d_logits)))

    def naive_prefill(self, framed_chunks, query_tokens, mode: MaskMode, counter: FlopCounter | None = None,
                      keep_context: bool = True):
        chunks = [np.asarray(c, np.int32) for c in framed_chunks]
        flat = _i32(np.concatenate(chunks) if chunks else np.zeros(0))
        offs = np.ascontiguousarray(np.concatenate([[0], np.cumsum([len(c) for c in chunks])]), np.int64)
        q = _i32(query_tokens)
        out = np.zeros(self.config.vocab_size, np.float32)
        fl = _Flops()
        h = C.c_void_p()
        _check(lib().tkv_naive_prefill(self._h, _p(flat, I32P), _p(offs, I64P), len(chunks),
                                       _p(q, I32P) if len(q) else None, len(q), int(mode), _p(out, F32P),
                                       C.byref(fl), C.byref(h) if keep_context else None))
        if counter is not None:
            counter._add(fl)
        return AssembledContext(self, h) if keep_context else out[None, :]

    def naive_prefill_ids(self, chunk_ids, query_tokens, mode: MaskMode, counter: FlopCounter | None = None):
        ids = np.ascontiguousarray(np.asarray(list(chunk_ids), dtype=np.uint64))
        q = _i32(query_tokens)
        out = np.zeros(self.config.vocab_size, np.float32)
        fl = _Flops()
        h = C.c_void_p()
        _check(lib().tkv_naive_prefill_ids(self._h, _p(ids, U64P) if len(ids) else None, len(ids),
                                           _p(q, I32P) if len(q) else None, len(q), int(mode), _p(out, F32P),
                                           C.byref(fl), C.byref(h)))
        if counter is not None:
            counter._add(fl)
        return AssembledContext(self, h)

    def greedy_decode(self, ctx: AssembledContext, max_new: int, eos: int = EOS) -> list[int]:
        out = np.zeros(max(max_new, 1), np.int32)
        n = C.c_int64()
        _check(lib().tkv_greedy_decode(self._h, ctx.handle, max_new, _p(out, I32P), C.byref(n)))
        return out[:n.value].tolist()

    # ---- multi-GPU store sharding (include/tkv.h, "Multi-GPU") ----
    def export_ipc(self) -> bytes:
        h = _Ipc()
        _check(lib().tkv_store_export_ipc(self._h, C.byref(h), None))
        return bytes(h.bytes)

    def attach_ipc(self, slot: int, handle: bytes) -> None:
        h = _Ipc()
        C.memmove(h.bytes, handle, 64)
        _check(lib().tkv_store_attach_ipc(self._h, slot, C.byref(h)))

    def store_rebalance(self, max_moves: int = 1 << 30) -> tuple[int, int]:
        """tkv_store_rebalance: frequency-driven HBM <-> host tier moves; returns (promoted, demoted)."""
        up, down = C.c_int64(), C.c_int64()
        _check(lib().tkv_store_rebalance(self._h, max_moves, C.byref(up), C.byref(down)))
        return up.value, down.value

    def export_directory(self) -> bytes:
        """tkv_store_export_directory: this engine's owned chunks + pool IPC handle + identity, as one blob."""
        n = C.c_int64()
        _check(lib().tkv_store_export_directory(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(max(n.value, 1))
        _check(lib().tkv_store_export_directory(self._h, buf, n.value, C.byref(n)))
        return buf.raw[:n.value]

    def import_directory(self, slot: int, blob: bytes) -> None:
        """tkv_store_import_directory: validate a peer's blob and register its chunks under peer slot `slot`."""
        _check(lib().tkv_store_import_directory(self._h, slot, blob, len(blob)))

    def attach_engine(self, slot: int, peer: "Engine") -> None:
        _check(lib().tkv_store_attach_engine(self._h, slot, peer.handle))

    def chunk_pages(self, chunk_id: int):
        n, ln = C.c_int64(), C.c_int64()
        _check(lib().tkv_store_chunk_pages(self._h, chunk_id, None, 0, C.byref(n), C.byref(ln)))
        pages = np.zeros(max(n.value, 1), np.int32)
        _check(lib().tkv_store_chunk_pages(self._h, chunk_id, _p(pages, I32P), len(pages), C.byref(n), C.byref(ln)))
        return pages[:n.value], ln.value

    def register_remote(self, chunk_id: int, slot: int, length: int, pages, framed=None) -> None:
        pages = _i32(pages)
        fr = _i32(framed) if framed is not None else None
        _check(lib().tkv_store_register_remote(self._h, chunk_id, slot, length, _p(pages, I32P), len(pages),
                                               _p(fr, I32P) if fr is not None else None))

    def fetch_remote(self, chunk_id: int) -> None:
        _check(lib().tkv_store_fetch_remote(self._h, chunk_id))

    def remote_bytes(self) -> int:
        return lib().tkv_remote_bytes(self._h)

    # ---- measurement ----
    def stream_ptr(self) -> int:
        return lib().tkv_engine_stream(self._h) or 0

    def profile(self, on: bool) -> None:
        _check(lib().tkv_profile_enable(self._h, int(on)))

    def profile_reset(self) -> None:
        _check(lib().tkv_profile_reset(self._h))

    def profile_read(self, kernel_class: str):
        ms, n = C.c_double(), C.c_int64()
        _check(lib().tkv_profile_read(self._h, kernel_class.encode(), C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def launch_count(self) -> int:
        return lib().tkv_launch_count(self._h)

    def io_bytes(self) -> tuple[int, int]:
        """(host->device, device->host) bytes copied by the engine since creation."""
        h, d = C.c_int64(), C.c_int64()
        _check(lib().tkv_io_bytes(self._h, C.byref(h), C.byref(d)))
        return h.value, d.value

    TIMELINE_CLASSES = ("gather_rope", "attention", "gemm", "epilogue", "other")

    def kernel_timeline(self, on: bool):
        """tkv_kernel_timeline: arm (on=True) / read (on=False) the in-chain kernel timeline; returns
        ([launches][2] globaltimer ns = (first CTA past griddepcontrol.wait, last warp done), [launches] class index
        into TIMELINE_CLASSES) in stream order."""
        if on:
            _check(lib().tkv_kernel_timeline(self._h, 1, None, None, 0, None))
            return None
        cap = 8192
        buf = np.zeros(2 * cap, np.uint64)
        cls = np.zeros(cap, np.int32)
        n = C.c_int64()
        _check(lib().tkv_kernel_timeline(self._h, 0, buf.ctypes.data_as(U64P), cls.ctypes.data_as(I32P), cap,
                                         C.byref(n)))
        m = min(n.value, cap)
        return buf[:2 * m].reshape(-1, 2).astype(np.int64), cls[:m].copy()

    def set_mask_rows(self, rows, lo, hi) -> None:
        """Override mask rows of the next naive prefill (testing::mask_fault_hook): row r sees keys [lo, hi]."""
        r = np.ascontiguousarray(rows, np.int64)
        a, b = _i32(lo), _i32(hi)
        _check(lib().tkv_debug_set_mask_rows(self._h, _p(r, I64P), _p(a, I32P), _p(b, I32P), len(r)))

    def set_mask_fault(self, row: int, col: int) -> None:
        _check(lib().tkv_debug_set_mask_fault(self._h, row, col))


def debug_gemm(A: np.ndarray, W: np.ndarray, dtype: str = "bf16", use_tc: bool = True, splits: int = 1,
               device: int = 0) -> np.ndarray:
    """out = A . W^T through the engine's GEMM kernel (kernel unit tests)."""
    A = np.ascontiguousarray(A, np.float32)
    W = np.ascontiguousarray(W, np.float32)
    M, K = A.shape
    N = W.shape[0]
    out = np.zeros((M, N), np.float32)
    dt = Dtype.F32 if dtype == "f32" else Dtype.BF16
    _check(lib().tkv_debug_gemm(device, int(dt), int(use_tc), _p(A, F32P), _p(W, F32P), M, N, K, splits,
                                _p(out, F32P)))
    return out


def embed(tokens, dim: int = 256) -> np.ndarray:
    """embed (retrieval.cpp:64-88)."""
    t = _i32(tokens)
    out = np.zeros(dim, np.float64)
    _check(lib().tkv_embed(_p(t, I32P) if len(t) else None, len(t), dim, out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def debug_attention(q, k, v, lo, hi, H: int, Hkv: int, d: int, dtype: str = "bf16", impl: int = 0,
                    device: int = 0) -> np.ndarray:
    """The engine's flash attention with the [lo, hi] row predicate (kernel unit tests)."""
    q = np.ascontiguousarray(q, np.float32)
    k = np.ascontiguousarray(k, np.float32)
    v = np.ascontiguousarray(v, np.float32)
    lo = _i32(lo)
    hi = _i32(hi)
    Tq, Tk = q.shape[0], k.shape[0]
    out = np.zeros((Tq, H * d), np.float32)
    dt = Dtype.F32 if dtype == "f32" else Dtype.BF16
    _check(lib().tkv_debug_attention(device, int(dt), impl, _p(q, F32P), _p(k, F32P), _p(v, F32P), _p(lo, I32P),
                                     _p(hi, I32P), Tq, Tk, H, Hkv, d, _p(out, F32P)))
    return out


def greedy_decode(engine: Engine, ctx: AssembledContext, max_new: int, eos: int = EOS) -> list[int]:
    """model.hpp:74-81"""
    return engine.greedy_decode(ctx, max_new, eos)
