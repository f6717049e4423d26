"""CPU: the C-ABI library builds for sm_100a, loads without a GPU, and exports
exactly the entry points include/taco.h declares (each bound in _lib)."""

import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "taco.h")


def _declared() -> set[str]:
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(taco_[a-z0-9_]+)\s*\(", text))


def test_header_declares_the_hot_path_entry_points():
    names = _declared()
    for want in ("taco_row_update", "taco_construct", "taco_tour_cost", "taco_elite_order",
                 "taco_elite_neighbors", "taco_select_parity", "taco_selection_table"):
        assert want in names


def test_library_exports_every_declared_symbol(built_lib):
    out = subprocess.run(["nm", "-D", "--defined-only", built_lib], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (taco_[a-z0-9_]+)$", out, flags=re.M))
    assert _declared() <= exported, _declared() - exported


def test_library_is_sm100a(built_lib):
    out = subprocess.run(["cuobjdump", "--list-elf", built_lib], capture_output=True, text=True).stdout
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out


def test_ctypes_binding_covers_the_header(built_lib):
    from paper_2404_04895_b200 import _lib

    assert set(_lib.SIGNATURES) == _declared()
    lib = _lib.load(built_lib)
    assert lib.taco_abi_version() == _lib.ABI_VERSION
    assert lib.taco_status_string(_lib.TACO_NO_CANDIDATE) == b"selector chose a visited city"
    assert lib.taco_max_sorted_n() >= 10000


def test_bad_arguments_are_rejected_without_a_gpu(built_lib):
    # argument validation happens before any CUDA call
    from paper_2404_04895_b200 import _lib

    lib = _lib.load(built_lib)
    assert lib.taco_construct(2, 1, 0, 0, None, 0, None, None, 0, 0, None, None, None, None, None,
                              None, 1.0, None, 1.0, None, None) == _lib.TACO_ERR_ARG
    # a fallback multiplier without its base
    assert lib.taco_construct(10, 1, 0, 0, None, 32, None, None, 0, 0, None, 8, None, None, None,
                              None, 1.0, 8, 1.0, None, None) == _lib.TACO_ERR_ARG
    assert lib.taco_row_update(2, None, None, None, None, None, 0, None, None, 0, 1.0, 0, 1.0, 1.0,
                               None, None, None, 0, None, None, None, None, None) == _lib.TACO_ERR_ARG
    assert lib.taco_construct_rw(3, 1, 0, None, 0, 0, None, None, None, None, None, 0, None,
                                 None) == _lib.TACO_ERR_ARG
    assert lib.taco_iter_advance(None, None, 1, None) == _lib.TACO_ERR_ARG
    assert lib.taco_coord_instance(2, None, 0, None, None, 0, None, None) == _lib.TACO_ERR_ARG
    assert lib.taco_log_weights(10, None, 0.0, None, None) == _lib.TACO_ERR_ARG
    with pytest.raises(ValueError):
        _lib.check(_lib.TACO_ERR_ARG, "x")


def test_product_path_fails_loudly_without_cuda(monkeypatch):
    import torch

    import paper_2404_04895_b200 as taco
    from paper_2404_04895_b200 import _device

    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    inst = taco.euclidean_instance([[0, 0], [1, 0], [0, 1], [1, 1]])
    with pytest.raises(_device.NoCudaDevice):
        taco.compute_probability_matrix(taco.PheromoneState.initial(4, 1.0), inst, taco.AcoParams(m=2, k=1))
    with pytest.raises(_device.NoCudaDevice):
        taco.Solver(inst, n_ants=2)
