"""GPU: TKVW weights files (docs/formats.md "TKVW"; save_weights / load_weights, proj/src/model.cpp:120-196) through
the engine, against the UNMODIFIED reference: files are byte-identical both ways, an engine loaded from a file carries
the reference fingerprint and the seeded engine's exact logits, damaged files fail like load_weights
(proj/tests/test_model.cpp:93-139), and weights that are NOT init_random's (non-unit RMSNorm weights) run the
reference's own forward_tokens numbers."""
import struct

import numpy as np
import pytest

import oracle as O
from paper_2410_07590_b200 import turbokv as T
from tests.test_gpu_parity import BF16_TOL, FP32_TOL, assert_close

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.Ref.available(), reason="reference library not built")]


def ref_save(cfg: O.Cfg, seed: int, path) -> None:
    O.Ref.check(O.Ref.lib().ref_save_weights(cfg.c(), seed, str(path).encode()))


@pytest.mark.parametrize("name,cfg", [("toy", O.TOY), ("qwen1", O.qwen_layers(1))])
def test_save_weights_byte_identical_to_reference(tmp_path, name, cfg):
    ours, theirs = tmp_path / "ours.tkvw", tmp_path / "ref.tkvw"
    T.save_weights(T.ModelConfig(**vars(cfg)), 42, ours)
    ref_save(cfg, 42, theirs)
    assert ours.read_bytes() == theirs.read_bytes()
    c, ck = O.OracleCfg(), O.C.c_uint64()
    O.Ref.check(O.Ref.lib().ref_load_weights(str(ours).encode(), O.C.byref(c), O.C.byref(ck)))  # reference accepts it
    assert ck.value == O.Ref.identity(cfg, 42)[0]


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_engine_from_reference_weights_file(tmp_path, golden, dtype):
    meta, A = golden
    m = meta["c1"]
    path = tmp_path / "toy.tkvw"
    ref_save(O.TOY, 42, path)
    eng = T.Engine(None, 0, dtype=dtype, store_capacity_tokens=4096, weights_path=path)
    seeded = T.Engine(T.ModelConfig.toy(), 42, dtype=dtype, store_capacity_tokens=4096)
    try:
        assert vars(eng.config) == vars(T.ModelConfig.toy())
        assert f"{eng.fingerprint():016x}" == m["fingerprint"]  # chunk ids = the reference engine's
        offs = A["c1.payload_offsets"]
        pays = [A["c1.payloads"][offs[i]:offs[i + 1]] for i in range(len(offs) - 1)]
        out = []
        for e in (eng, seeded):
            ids = e.ingest_chunks(pays)
            assert [f"{i:016x}" for i in ids] == m["ids"]
            with e.assemble(ids, T.PositionMode.Reordered) as ctx:
                out.append(e.prefill_query(ctx, A["c1.query"]).copy())
        assert np.array_equal(out[0], out[1])  # the same f64 values -> the same canonical cast -> the same logits
    finally:
        eng.close()
        seeded.close()


def test_damaged_weights_files_rejected(tmp_path):
    path = tmp_path / "w.tkvw"
    T.save_weights(T.ModelConfig.toy(), 42, path)
    raw = bytearray(path.read_bytes())
    flipped = bytearray(raw)
    flipped[100000] ^= 0x5A  # proj/tests/test_model.cpp:116-126
    (tmp_path / "flip.tkvw").write_bytes(bytes(flipped))
    with pytest.raises(T.FormatError, match="checksum"):
        T.Engine(None, 0, dtype="f32", store_capacity_tokens=256, weights_path=tmp_path / "flip.tkvw")
    bad = bytearray(raw)
    bad[:4] = b"NOPE"
    (tmp_path / "magic.tkvw").write_bytes(bytes(bad))
    with pytest.raises(T.FormatError, match="not a weights file"):
        T.Engine(None, 0, dtype="f32", store_capacity_tokens=256, weights_path=tmp_path / "magic.tkvw")
    (tmp_path / "short.tkvw").write_bytes(bytes(raw[:len(raw) // 2]))
    with pytest.raises(T.FormatError, match="truncated"):
        T.Engine(None, 0, dtype="f32", store_capacity_tokens=256, weights_path=tmp_path / "short.tkvw")
    with pytest.raises(T.NotFoundError):
        T.Engine(None, 0, dtype="f32", store_capacity_tokens=256, weights_path=tmp_path / "absent.tkvw")


def fnv_words(buf: bytes, h: int = 0xCBF29CE484222325) -> int:
    for b in buf:
        h = ((h ^ b) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


@pytest.mark.parametrize("dtype,tol", [("f32", FP32_TOL), ("bf16", BF16_TOL)])
def test_non_unit_norm_weights_match_reference_forward(tmp_path, dtype, tol):
    """A TKVW file whose RMSNorm weights are NOT 1.0 (every attn_norm / mlp_norm / final_norm rescaled): the engine's
    vanilla causal prefill equals the reference's forward_tokens over the same file."""
    cfg = O.TOY
    src = tmp_path / "src.tkvw"
    ref_save(cfg, 9, src)
    raw = bytearray(src.read_bytes())
    H, I, V, L = cfg.hidden_size, cfg.intermediate_size, cfg.vocab_size, cfg.layer_num
    qd, kvd = cfg.head_num * cfg.head_size, cfg.kv_dim
    at = 4 + 4 + 7 * 8 + 2 * 8  # header
    rng = np.random.default_rng(3)

    def skip_mat(at, r, c):
        assert struct.unpack_from("<QQ", raw, at) == (r, c)
        return at + 16 + 8 * r * c

    def scale_vec(at):
        (n,) = struct.unpack_from("<Q", raw, at)
        v = np.frombuffer(raw, np.float64, n, at + 8).copy() * rng.uniform(0.5, 1.5, n)
        raw[at + 8:at + 8 + 8 * n] = v.tobytes()
        return at + 8 + 8 * n

    tensor_start = at
    at = skip_mat(at, V, H)
    for _ in range(L):
        at = scale_vec(at)
        at = scale_vec(at)
        for r, c in ((H, qd), (H, kvd), (H, kvd), (qd, H), (H, I), (H, I), (I, H)):
            at = skip_mat(at, r, c)
    at = scale_vec(at)
    at = skip_mat(at, H, V)
    raw[at:at + 8] = struct.pack("<Q", fnv_words(bytes(raw[tensor_start:at])))
    path = tmp_path / "norms.tkvw"
    path.write_bytes(bytes(raw))
    q = O.random_text_tokens(5, 40)
    ref = np.zeros(V)
    O.Ref.check(O.Ref.lib().ref_forward_file(str(path).encode(), q.ctypes.data_as(O.I32P), len(q),
                                             ref.ctypes.data_as(O.F64P)))
    eng = T.Engine(None, 0, dtype=dtype, store_capacity_tokens=256, weights_path=path)
    try:
        got = eng.naive_prefill([], q, T.MaskMode.Causal, keep_context=False)[0]
        assert_close(got, ref, tol)
        base = T.Engine(T.ModelConfig.toy(), 9, dtype=dtype, store_capacity_tokens=256)
        plain = base.naive_prefill([], q, T.MaskMode.Causal, keep_context=False)[0]
        base.close()
        assert np.abs(plain - got).max() > 1e-3  # the norm weights really are in use
    finally:
        eng.close()
