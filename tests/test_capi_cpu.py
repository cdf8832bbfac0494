"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every symbol include/tw_c.h declares, refuses to run without a CUDA device
(no CPU fallback), and the product package never touches the oracle."""
import os
import re

import numpy as np
import pytest

from paper_2211_04045_b200 import capi, scenes as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "tw_c.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tw_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = capi.lib()
    names = declared_symbols()
    assert len(names) >= 15
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(capi.EXPORTS)
    assert L.tw_abi_version() == 1


def test_default_config_matches_reference_defaults():  # resolve.hpp:13-34
    c = capi.make_config()
    assert (c.step_limit, c.eps, c.d_min, c.d_max, c.delta, c.sigma, c.gamma) == (512, 1e-4, 2e-3, 4e-3, 1e-3, 1.1, 0.9)
    assert (c.solver, c.sweeps, c.under_relax, c.family, c.edge_constraints) == (0, 1, 0.5, 0, 1)
    assert c.color_seed == 0x5EED
    with pytest.raises(ValueError):
        capi.make_config(bogus=1)


def _has_gpu():
    import ctypes

    try:
        cu = ctypes.CDLL("libcuda.so.1")
        n = ctypes.c_int(0)
        return cu.cuInit(0) == 0 and cu.cuDeviceGetCount(ctypes.byref(n)) == 0 and n.value > 0
    except OSError:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device behaviour")
def test_no_cpu_fallback_without_device():
    with pytest.raises(capi.TwError) as e:
        capi.Context(0)
    assert e.value.code == capi.TW_ECUDA


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2211_04045_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "pyoracle" not in txt and "liboracle" not in txt and "oracle.h" not in txt, f


def test_finalize_edges_matches_oracle():
    import pyoracle as O

    for sc in S.scene_fixtures(0):
        e = O.finalize_edges(sc.nv, np.zeros((0, 2)), sc.strand_edges, sc.triangles)
        assert np.array_equal(e, sc.edges), sc.name


def test_knot_scene_sizes():
    reef = S.knot_scene(n_along=935)
    assert reef.nv == 37400 and len(reef.triangles) == 70984 and len(reef.edges) == 108382
    bow = S.knot_scene(n_along=1870)
    assert bow.nv == 74800 and len(bow.triangles) == 142044


def test_small_knot_start_is_intersection_free():
    import pyoracle as O

    sc = S.knot_scene(n_along=150, n_across=8, pull=7e-3)
    assert O.ccd_certify(sc, sc.x, sc.x)[0] == 0
    assert O.ccd_certify(sc, sc.x, sc.y)[1] > 0  # the target penetrates
    sc = S.ply_knot(n_along=400, n_across=6)
    assert O.ccd_certify(sc, sc.x, sc.x)[0] == 0
