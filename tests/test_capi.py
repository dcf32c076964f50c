"""The C ABI without a GPU: libkpgemm.so loads, exports every symbol include/kpgemm.h
declares, and its host-only entry points (registry, dispatch tables, error codes)
behave.  The dispatch table must route exactly like predict_tree (classify.py:230-237)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT
from paper_2008_13145_b200 import _lib
from paper_2008_13145_b200.classify import TREE_PRESETS, predict_tree, predict_tree_batch, train_tree
from paper_2008_13145_b200.dataset import DEFAULT_WG_PAIRS, KernelConfig, ProblemSize, enumerate_configs
from paper_2008_13145_b200.selection import ConfigSubset

HEADER = (ROOT / "include" / "kpgemm.h").read_text()


def declared_symbols():
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(kp_\w+)\s*\(", HEADER, re.M)))


@pytest.fixture(scope="module")
def lib():
    return _lib.load()


def test_every_declared_symbol_is_exported(lib):
    syms = declared_symbols()
    assert len(syms) >= 16
    for name in syms:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} missing from the ctypes binding"


def test_registry_order_is_enumerate_configs(lib):
    assert lib.kp_abi_version() == 1
    for fam in (_lib.FAMILY_PAPER, _lib.FAMILY_SIMT):
        assert lib.kp_family_size(fam) == 640
        for idx, cfg in enumerate(enumerate_configs()):
            vid = lib.kp_family_variant(fam, idx)
            assert lib.kp_find_variant(fam, _lib.KernelChoice(*cfg.as_tuple())) == vid
            ch = _lib.KernelChoice()
            f = ctypes.c_int()
            assert lib.kp_variant_info(vid, ctypes.byref(ch), ctypes.byref(f)) == 0
            assert ch.as_tuple() == cfg.as_tuple() and f.value == fam


def test_error_codes_and_messages(lib):
    assert lib.kp_find_variant(_lib.FAMILY_SIMT, _lib.KernelChoice(3, 1, 1, 8, 8)) == _lib.KP_ENOENT
    assert b"no config" in lib.kp_last_error()
    assert lib.kp_family_size(99) == _lib.KP_EINVAL
    with pytest.raises(KeyError):
        _lib.check(lib.kp_variant_info(10 ** 6, None, None), "x")
    # shape validation happens before any CUDA call
    assert lib.kp_gemm(0, 0, 4, 4, 1, 8, 4, 0, 8, 4, 0, 8, 4, 0, None) == _lib.KP_EINVAL
    assert lib.kp_gemm(0, 4, 4, 4, 1, None, 4, 0, 8, 4, 0, 8, 4, 0, None) == _lib.KP_EINVAL
    assert lib.kp_gemm(0, 4, 8, 4, 1, 8, 4, 0, 8, 4, 0, 8, 4, 0, None) == _lib.KP_EINVAL  # lda < k
    with pytest.raises(ValueError):
        _lib.check(_lib.KP_EINVAL, "x")
    with pytest.raises(RuntimeError):
        _lib.check(_lib.KP_EIO, "x")


def _random_tree(seed, n_classes=5, rows=300):
    rng = np.random.default_rng(seed)
    feats = np.log2(rng.integers(1, 1 << 14, size=(rows, 4)).astype(np.float64))
    labels = rng.integers(0, n_classes, size=rows)
    return train_tree(feats, labels, TREE_PRESETS["A"], n_classes=n_classes)


def _load(lib, tree, variants):
    arrs = [np.ascontiguousarray(a, dtype=t) for a, t in ((tree.feature, np.int32), (tree.threshold, np.float64),
                                                          (tree.left, np.int32), (tree.right, np.int32),
                                                          (tree.leaf_class, np.int32))]
    c2v = np.ascontiguousarray(variants, dtype=np.int32)
    ptrs = [a.ctypes.data_as(ctypes.POINTER(ctypes.c_double if a.dtype == np.float64 else ctypes.c_int32))
            for a in arrs]
    return lib.kp_dispatch_load(tree.n_nodes, *ptrs, len(c2v), c2v.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_c_table_routes_like_predict_tree(lib, seed):
    tree = _random_tree(seed)
    variants = [lib.kp_family_variant(_lib.FAMILY_SIMT, i * 7) for i in range(5)]
    h = _load(lib, tree, variants)
    assert h >= 0
    rng = np.random.default_rng(100 + seed)
    dims = rng.integers(1, 1 << 15, size=(20000, 4))
    feats = np.log2(dims.astype(np.float64))
    want = predict_tree_batch(tree, feats)
    got = np.empty(len(feats), dtype=np.int64)
    buf = np.empty(4, dtype=np.float64)
    p = buf.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    for i, f in enumerate(feats):
        buf[:] = f
        got[i] = lib.kp_dispatch_class_feats(h, p)
    assert np.array_equal(got, want)
    # variant ids through the class map, and the C-log2 convenience entry point
    for i in range(0, 2000, 97):
        buf[:] = feats[i]
        assert lib.kp_dispatch_select_feats(h, p) == variants[want[i]]
        m, k, n, b = (int(v) for v in dims[i])
        assert lib.kp_dispatch_select(h, m, k, n, b) == variants[predict_tree(tree, np.log2([m, k, n, b]))]
    assert lib.kp_dispatch_free(h) == 0
    assert lib.kp_dispatch_class_feats(h, p) == _lib.KP_ENOENT


def test_dispatch_load_rejects_malformed_trees(lib):
    tree = _random_tree(5, n_classes=3)
    good = [lib.kp_family_variant(_lib.FAMILY_PAPER, i) for i in range(3)]
    assert _load(lib, tree, [good[0], good[1], 10 ** 6]) == _lib.KP_ENOENT
    bad = type(tree)(tree.feature, tree.threshold, tree.left.copy(), tree.right, tree.leaf_class)
    internal = int(np.flatnonzero(tree.leaf_class < 0)[0])
    bad.left[internal] = 0  # cycle back to the root
    assert _load(lib, bad, good) == _lib.KP_EINVAL
    assert b"not a tree" in lib.kp_last_error() or b"reachable" in lib.kp_last_error()
    assert _load(lib, tree, good[:2]) == _lib.KP_EINVAL  # leaf class outside the class map


def test_k_slice_plan_host_logic(lib):
    """kp_gemm_plan with an explicit SM count needs no GPU.  SIMT rule (fitted on measured
    forced-S data): tiles per SM u < 0.15 -> 16 slices, < 0.5 -> 8, < 2 -> 4, < 6 -> 2, else 1,
    halved while the grid would exceed 4 waves of resident CTAs, never shallower than 64
    in k; no empty slice, k-tile aligned; the paper family and a cap of 1 never slice."""
    from paper_2008_13145_b200 import gemm
    probs = [ProblemSize(196, 4608, 512, 1), ProblemSize(32, 25088, 4096, 1), ProblemSize(1, 4096, 1000, 1),
             ProblemSize(12544, 4608, 512, 1), ProblemSize(3136, 2304, 256, 1), ProblemSize(50, 300, 70, 4),
             ProblemSize(64, 255, 64, 1), ProblemSize(7, 100000, 9, 1), ProblemSize(784, 512, 128, 1)]
    seen_sliced = 0
    for cfg in enumerate_configs()[::7]:
        tiles_m, tiles_n = cfg.tile_rows * cfg.wg_rows, cfg.tile_cols * cfg.wg_cols
        for p in probs:
            s, kps = gemm.k_slice_plan(cfg, p, num_sms=148)
            assert 1 <= s <= 16  # 16/8/4/2, fewer when k has fewer k-tiles than that
            if s == 1:
                assert kps == p.k
                continue
            seen_sliced += 1
            assert p.k // s >= 64 and kps >= 64
            assert (s - 1) * kps < p.k <= s * kps  # no empty slice
            assert kps % 8 == 0  # a whole number of k-tiles (BK in {8, 16, 32})
            tiles = -(-p.m // tiles_m) * -(-p.n // tiles_n) * p.batch
            assert tiles < (0.15 if s > 8 else 0.5 if s > 4 else 2 if s > 2 else 6) * 148  # tiles-per-SM bins
        big = ProblemSize(16384, 4096, 16384, 1)
        assert gemm.k_slice_plan(cfg, big, num_sms=148) == (1, 4096)
        assert gemm.k_slice_plan(cfg, ProblemSize(1, 4096, 1, 1), family="paper", num_sms=148) == (1, 4096)
    assert seen_sliced > 50
    prev = gemm.set_max_k_slices(1)
    try:
        assert gemm.k_slice_plan(KernelConfig(4, 8, 8, 16, 8), probs[0], num_sms=148) == (1, 4608)
    finally:
        assert gemm.set_max_k_slices(prev) == 1
    assert lib.kp_set_max_k_slices(0) == _lib.KP_EINVAL


def test_simt_staging_switch(lib):
    from paper_2008_13145_b200 import gemm

    """kp_set_simt_staging: 1 (TMA, default) / 0 (cp.async), previous mode returned."""
    assert gemm.set_simt_staging("cp.async") == "tma"
    try:
        assert gemm.set_simt_staging("cp.async") == "cp.async"
    finally:
        assert gemm.set_simt_staging("tma") == "cp.async"
    assert lib.kp_set_simt_staging(2) == _lib.KP_EINVAL
    assert lib.kp_set_simt_staging(-1) == _lib.KP_EINVAL
    with pytest.raises(ValueError):
        gemm.set_simt_staging("ldgsts")


def test_operand_repack_switch(lib):
    """kp_set_operand_repack: 1 (repack unaligned rows when it pays, default) / 2 (always)
    / 0 (never: in-kernel staging); the previous mode is returned."""
    from paper_2008_13145_b200 import gemm
    assert gemm.set_operand_repack("always") == "auto"
    try:
        assert gemm.set_operand_repack("never") == "always"
    finally:
        assert gemm.set_operand_repack("auto") == "never"
    assert lib.kp_set_operand_repack(3) == _lib.KP_EINVAL
    assert lib.kp_set_operand_repack(-1) == _lib.KP_EINVAL
    with pytest.raises(ValueError):
        gemm.set_operand_repack("sometimes")


def test_conv3x3_supported_query(lib):
    """kp_conv3x3_supported needs no GPU: SIMT variants with TMA staging and C a multiple
    of their k-tile depth, TF32 variants with C % 32 == 0, BF16 variants with C % 64 == 0
    and Cout % 8 == 0; never the paper family; bad ids -ENOENT."""
    from paper_2008_13145_b200 import gemm
    vid = gemm.variant_id(KernelConfig(8, 8, 8, 16, 8), "simt")
    assert lib.kp_conv3x3_supported(vid, 64, 64) == 1
    assert lib.kp_conv3x3_supported(vid, 3, 64) == 0
    assert lib.kp_conv3x3_supported(vid, 64, 62) == 0
    assert lib.kp_conv3x3_supported(gemm.variant_id(KernelConfig(8, 8, 8, 1, 128), "simt"), 64, 64) == 0  # BN 1024
    assert lib.kp_conv3x3_supported(gemm.variant_id(KernelConfig(8, 8, 8, 16, 8), "paper"), 64, 64) == 0
    assert lib.kp_conv3x3_supported(10 ** 6, 64, 64) == _lib.KP_ENOENT
    for cfg in gemm.family_configs("tf32"):
        tid = gemm.variant_id(cfg, "tf32")
        assert lib.kp_conv3x3_supported(tid, 64, 64) == 1
        assert lib.kp_conv3x3_supported(tid, 48, 64) == 0  # not a whole 32-channel slab
        assert lib.kp_conv3x3_supported(tid, 64, 62) == 0
    for cfg in gemm.family_configs("bf16"):
        bid = gemm.variant_id(cfg, "bf16")
        assert lib.kp_conv3x3_supported(bid, 64, 64) == 1
        assert lib.kp_conv3x3_supported(bid, 32, 64) == 0  # not a whole 64-channel slab
        assert lib.kp_conv3x3_supported(bid, 64, 60) == 0  # weight rows not 16-byte pitched
