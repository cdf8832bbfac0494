"""The reference's C++ stage API (include/twoway/{distance,proximity,
constraints,advance,resolve}.hpp) called the way a reference caller calls it
(tests/cpp/stage_api_probe.cpp, compiled here against the in-tree library),
compared with the oracle bit for bit: proximity_search, refresh_distances,
linearize_all, color_constraints (reference coloring), advance, resolve."""
import os
import subprocess

import numpy as np
import pytest

import pyoracle as O
from paper_2211_04045_b200 import scenes as S

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2211_04045_b200")


@pytest.fixture(scope="module")
def probe(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("probe") / "stage_api_probe")
    subprocess.run(["g++", "-O2", "-std=c++20", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "stage_api_probe.cpp"), "-o", exe, "-L" + PKG,
                    "-l:libtwoway_b200.so", "-Wl,-rpath," + PKG], check=True)
    return exe


def _bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


class _Reader:
    def __init__(self, b):
        self.b, self.o = b, 0

    def take(self, dtype, n):
        a = np.frombuffer(self.b, dtype=dtype, count=n, offset=self.o)
        self.o += a.nbytes
        return a


def _cases():
    return [sc for sc in S.scene_fixtures(0) if len(sc.triangles) and not len(sc.strand_edges)][:8]


@pytest.mark.parametrize("sc", _cases(), ids=lambda s: s.name)
def test_cpp_stage_api_matches_oracle(probe, tmp_path, sc):
    x, y = np.asarray(sc.x, np.float64), np.asarray(sc.y, np.float64)
    inv = np.asarray(sc.inv_mass, np.float64)
    tris = np.asarray(sc.triangles, np.int32)
    fin, fout = tmp_path / "in.bin", tmp_path / "out.bin"
    with open(fin, "wb") as f:
        f.write(np.array([len(x), len(tris)], np.int32).tobytes())
        f.write(x.tobytes() + y.tobytes() + inv.tobytes() + tris.tobytes())
    subprocess.run([probe, str(fin), str(fout)], check=True)
    r = _Reader(open(fout, "rb").read())
    nv = len(x)

    # proximity_search at y
    Py = O.search(sc, y, 4e-3)
    n = int(r.take(np.int64, 1)[0])
    rec = np.frombuffer(r.take(np.uint8, n * 16).tobytes(), dtype=[("k", np.uint64), ("d", np.float64)])
    assert n == len(Py)
    assert np.array_equal(rec["k"], Py.keys) and np.array_equal(_bits(rec["d"]), _bits(Py.dist))
    # refresh_distances at x
    Pr = Py.take(len(Py))
    O.refresh(sc, x, 4e-3, Pr)
    rr = np.frombuffer(r.take(np.uint8, n * 12).tobytes(), dtype=[("d", np.float64), ("a", np.int32)])
    assert np.array_equal(_bits(rr["d"]), _bits(Pr.dist))
    assert np.array_equal(rr["a"], (Pr.flags & 1).astype(np.int32))
    # linearize_all at y + reference coloring
    E = np.asarray(sc.edges).reshape(-1, 2)
    et = np.linalg.norm(x[E[:, 0]] - x[E[:, 1]], axis=1)
    Ro = O.linearize(sc, y, Py, et, delta=1e-3)
    nco, co = O.color(sc, Ro, 0x5EED, mode=0)
    nrows = int(r.take(np.int64, 1)[0])
    ncol = int(r.take(np.int64, 1)[0])
    assert nrows == len(Ro) and ncol == nco
    row = np.dtype([("head", np.int32, 4), ("verts", np.int32, 4), ("value", np.float64), ("diag", np.float64),
                    ("key", np.uint64), ("jac", np.float64, 12)])
    rows = np.frombuffer(r.take(np.uint8, nrows * row.itemsize).tobytes(), dtype=row)
    assert np.array_equal(rows["head"][:, 0], Ro.kind.astype(np.int32))
    assert np.array_equal(rows["head"][:, 1], Ro.nverts)
    assert np.array_equal(rows["head"][:, 3], co)
    contact = Ro.kind != O.ROW_EDGE
    assert np.array_equal(rows["key"][contact], Ro.pair_key[contact])
    assert np.array_equal(rows["head"][~contact, 2], Ro.edge_index[~contact])
    assert np.array_equal(_bits(rows["value"]), _bits(Ro.value))
    assert np.array_equal(_bits(rows["diag"]), _bits(Ro.diag))
    for i in range(nrows):
        k = Ro.nverts[i]
        assert np.array_equal(rows["verts"][i, :k], Ro.verts[i, :k])
        assert np.array_equal(_bits(rows["jac"][i, :3 * k]), _bits(Ro.jac[i, :k].reshape(-1)))
    # advance from x with the pair set at x
    Px = O.search(sc, x, 4e-3)
    D = O.vertex_bound(sc, 4e-3, Px, nv)
    xa, ra, md = O.advance(inv, y, D, 0.9, x, np.ones(nv))
    assert np.array_equal(_bits(r.take(np.float64, 3 * nv)), _bits(xa.reshape(-1)))
    assert np.array_equal(_bits(r.take(np.float64, nv)), _bits(ra))
    assert _bits(r.take(np.float64, 1))[0] == _bits(np.array([md]))[0]
    # resolve (device coloring, the ResolveConfig default)
    xo, st = O.resolve(sc, coloring_mode="device")
    assert np.array_equal(_bits(r.take(np.float64, 3 * nv)), _bits(xo.reshape(-1)))
    assert int(r.take(np.int32, 1)[0]) == st["steps"]
