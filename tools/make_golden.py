"""Generate the golden fixtures under tests/golden/ from the REAL reference.

The reference's own sources are compiled here against the Eigen-subset shim
(oracle/Makefile.ref -> oracle/_ref/libtwoway_ref.so). The
golden vectors are the reference's outputs on its own deterministic fixture
battery (testkit scene_fixtures(0), which scenes.scene_fixtures(0) reproduces
bit for bit -- asserted below). The device-coloring mode has no reference
counterpart; its vectors come from the C oracle's statement of the device
coloring. The script refuses to write when the C oracle disagrees with the
reference in reference mode. Files:

  resolve_fixtures.npz  per fixture and coloring mode: x_out (bits), steps,
                        searches, converged, final_residual, step_max_disp
  search_fixtures.npz   per fixture: sorted pair keys and distances of the
                        proximity search at x and at y (d_max = 4 mm)

usage: python tools/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import pyoracle as O  # noqa: E402
import pyref as R  # noqa: E402

from paper_2211_04045_b200 import scenes as S  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def main():
    os.makedirs(OUT, exist_ok=True)
    res, srch = {}, {}
    for i, sc in enumerate(S.scene_fixtures(0)):
        tag = f"{i:02d}_{sc.name}"
        name, rm, rx, ry, _, _ = R.fixture(i, 0)
        assert name == sc.name and np.array_equal(rx.view(np.uint64), sc.x.view(np.uint64)) \
            and np.array_equal(ry.view(np.uint64), sc.y.view(np.uint64)), tag
        for mode in ("reference", "device"):
            x, st = O.resolve(sc, coloring_mode=mode)
            if mode == "reference":
                xr, sr = R.resolve(rm, sc.x, sc.y)
                assert np.array_equal(xr.view(np.uint64), x.view(np.uint64)), tag
                assert np.array_equal(sr["step_max_disp"].view(np.uint64), st["step_max_disp"].view(np.uint64)), tag
                x, st = xr, sr
            p = f"{tag}/{mode}/"
            res[p + "x_out"] = x
            res[p + "stats"] = np.array([st["steps"], st["searches"], st["converged"], st["hit_step_limit"],
                                         st["start_in_contact"], st["step_law_violated"]], np.int64)
            res[p + "final_residual"] = np.array([st["final_residual"]])
            res[p + "step_max_disp"] = st["step_max_disp"]
        for where, pos in (("x", sc.x), ("y", sc.y)):
            keys, dist, _ = R.search(rm, pos, 4e-3)
            P = O.search(sc, pos, 4e-3)
            assert np.array_equal(P.keys, keys) and np.array_equal(P.dist.view(np.uint64), dist.view(np.uint64)), tag
            srch[f"{tag}/{where}/keys"] = keys
            srch[f"{tag}/{where}/dist"] = dist
    np.savez_compressed(os.path.join(OUT, "resolve_fixtures.npz"), **res)
    np.savez_compressed(os.path.join(OUT, "search_fixtures.npz"), **srch)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
