"""The C-ABI library: builds for sm_100a, loads on a CPU-only host, exports every entry point
include/cosine_verify.h declares, and fails cleanly (status codes, no crash) without a GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for f in os.listdir(os.path.join(ROOT, "include")):
        if f.endswith(".h"):
            src = open(os.path.join(ROOT, "include", f)).read()
            names |= set(re.findall(r"^\s*(?:cosine_status_t|const char\*|int32_t)\s+(cosine_\w+)\s*\(", src, re.M))
    return names


def test_header_declares_the_north_star_calls():
    d = _declared()
    for n in ("cosine_verify_init", "cosine_fuse_drafts", "cosine_verify_batch", "cosine_sample_residual"):
        assert n in d


def test_library_exports_every_declared_symbol():
    from paper_2503_10325_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for n in _declared():
        assert hasattr(lib, n), n
    assert set(_lib.EXPORTED_SYMBOLS) >= _declared()


def test_library_is_sm100a():
    import subprocess
    from paper_2503_10325_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_null_and_invalid_arguments_return_status_codes():
    from paper_2503_10325_b200 import _lib
    L = _lib._lib
    # NULL context -> INVALID_ARGUMENT, enqueues nothing, never crashes
    assert L.cosine_verify_batch(None, None, 1, 1, 1, None, 8, 1.0, None, 8, None, None, None, 0, 0, 0,
                                 None, None, None, None) == 1
    assert L.cosine_fuse_drafts(None, None, 1, 1, 1, None, 8, None, None, 0, 1.0, 0, 0, None, None, None,
                                None, 0, None) == 1
    assert L.cosine_sample_residual(None, None, 1, None, 8, 1.0, None, None, None, 8, None, None, 1, None,
                                    None, 0, None, None) == 1
    assert L.cosine_verify_destroy(None) == 0
    cfg = _lib.cosine_config_t(device=0, vocab_size=0, vocab_begin=0, vocab_end=0, max_batch=1, max_draft_len=1,
                               max_drafters=1, target_dtype=0, draft_dtype=0, draft_kind=0, seed=0, nranks=1,
                               rank=0, nccl_unique_id=None, cluster_size=0)
    h = ctypes.c_void_p()
    assert L.cosine_verify_init(ctypes.byref(cfg), ctypes.byref(h)) == 1
    assert b"vocabulary" in L.cosine_last_error(None)
    cfg.vocab_size, cfg.vocab_end, cfg.max_drafters = 100, 100, 9
    assert L.cosine_verify_init(ctypes.byref(cfg), ctypes.byref(h)) == 1
    cfg.max_drafters, cfg.exchange = 1, 7  # exchange must be 0 (automatic) or 1 (NCCL)
    assert L.cosine_verify_init(ctypes.byref(cfg), ctypes.byref(h)) == 1
    assert b"exchange" in L.cosine_last_error(None)
    # virtual groups: G >= 2, cfgs[g] must be rank g of G with tiling shards
    cfg.exchange = 0
    cfgs = (_lib.cosine_config_t * 2)(cfg, cfg)
    hs = (ctypes.c_void_p * 2)()
    assert L.cosine_verify_init_vgroup(cfgs, 1, hs) == 1
    assert L.cosine_verify_init_vgroup(cfgs, 2, hs) == 1  # nranks / rank / shards not set
    assert b"vgroup" in L.cosine_last_error(None)
    assert L.cosine_verify_batch_vgroup(None, 2, None, 1, 1, 1, None, 8, 1.0, None, 8, None, None, None, 0, 0,
                                        None, None, None, 0) == 1
    assert L.cosine_exchange_mode(None) == 0


def test_init_without_gpu_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2503_10325_b200 import _lib
    with pytest.raises(_lib.CosineError) as e:
        _lib.cosine_verify_init(1000, max_batch=2, max_draft_len=2, max_drafters=2)
    assert e.value.code == 3


def test_no_cpu_fallback_in_product_path():
    # the product package never imports the oracle (test infrastructure only)
    pkg = os.path.join(ROOT, "paper_2503_10325_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith(".py"):
                src = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", src, re.M), f
