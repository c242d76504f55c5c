"""CPU: the C-ABI library loads and exports every entry point include/tkv.h declares; host-side logic
(identity chain, presets, error mapping) matches the reference goldens; the header-only C++ shim
(include/turbokv_compat.hpp) compiles and links. No kernels run here."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2410_07590_b200 import turbokv as T

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "tkv.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tkv_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    lib = T.lib()
    names = declared_symbols()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.tkv_abi_version() == 2


def test_status_codes_mirror_reference_error_classes():
    # one code per turbokv::*Error (include/turbokv/errors.hpp:10-67)
    names = [T.lib().tkv_status_name(i).decode() for i in range(13)]
    assert names == ["ok", "error", "shape", "domain", "config", "degenerate_row", "io", "format", "not_found",
                     "stale_cache", "no_context", "cuda", "oom"]
    assert T._ERRORS[9] is T.StaleCacheError and T._ERRORS[5] is T.DegenerateRowError


def test_identity_chain_matches_goldens(golden):
    meta, A = golden
    ck, fp = T.weights_identity(T.ModelConfig.toy(), 42)
    assert (ck, fp) == (0x783FE06586F74DC9, 0x8DD32810BD252FD1)  # proj/docs/formats.md:107-112
    assert T.weights_identity(T.ModelConfig.toy(), 7)[0] == 0x37E1ED82918F7BBC
    offs = A["c1.payload_offsets"]
    for i, hexid in enumerate(meta["c1"]["ids"]):
        framed = T.frame_chunk(A["c1.payloads"][offs[i]:offs[i + 1]])
        assert f"{T.chunk_content_id(framed, fp):016x}" == hexid


def test_presets_and_validation():
    q = T.ModelConfig.qwen2_7b_like()
    assert (q.layer_num, q.head_num, q.kv_head_num, q.head_size, q.hidden_size, q.intermediate_size) == \
        (28, 28, 4, 128, 3584, 18944)  # proj/src/config.cpp:56-66
    with pytest.raises(T.ConfigError):
        T.ModelConfig.preset("nope")
    with pytest.raises(T.ConfigError):
        T.ModelConfig(4, 8, 3, 8, 64, 192, 259).validate()
    with pytest.raises(T.ConfigError):
        T.ModelConfig(4, 8, 2, 7, 56, 192, 259).validate()  # odd head_size
    assert T.ModelConfig.toy().fingerprint_seed() == T.ModelConfig.toy().fingerprint_seed()


@pytest.mark.skipif(__import__("tests.conftest", fromlist=["has_cuda"]).has_cuda(), reason="CPU-only check")
def test_no_cpu_fallback():
    with pytest.raises(T.CudaError):
        T.Engine(T.ModelConfig.toy(), 42)


def test_cpp_shim_compiles_and_links(tmp_path):
    exe = tmp_path / "compat_smoke"
    libdir = os.path.join(ROOT, "paper_2410_07590_b200")
    cmd = ["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "compat_smoke.cpp"),
           "-L", libdir, "-ltkv_b200", f"-Wl,-rpath,{libdir}", "-o", str(exe)]
    subprocess.run(cmd, check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "checksum 783fe06586f74dc9 fingerprint 8dd32810bd252fd1" in r.stdout


def test_embed_matches_reference():
    """tkv_embed (host side of the retrieval path) against the restatement and the reference itself."""
    import oracle as O

    for seed, n in ((1, 1), (2, 2), (3, 57), (4, 400)):
        t = O.random_text_tokens(seed, n)
        e = T.embed(t)
        assert np.array_equal(e, O.Port.embed(t))
        assert np.array_equal(e, O.Ref.embed(t))
    with pytest.raises(T.DomainError):
        T.embed([])
