"""Generate the golden fixtures under tests/golden/ from the C oracle.

The reference itself cannot be built here (Eigen is absent), so
the golden vectors are the oracle's outputs on the deterministic fixture
battery (scenes.scene_fixtures(0): the reference's acceptance fixtures plus
seeded random scenes). They pin the oracle against regressions and give the
GPU tests committed expectations:

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

from paper_2211_04045_b200 import scenes as S  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def main():
    os.makedirs(OUT, exist_ok=True)
    res, srch = {}, {}
    for i, sc in enumerate(S.scene_fixtures(0)):
        tag = f"{i:02d}_{sc.name}"
        for mode in ("reference", "device"):
            x, st = O.resolve(sc, coloring_mode=mode)
            p = f"{tag}/{mode}/"
            res[p + "x_out"] = x
            res[p + "stats"] = np.array([st["steps"], st["searches"], st["converged"], st["hit_step_limit"],
                                         st["start_in_contact"], st["step_law_violated"]], np.int64)
            res[p + "final_residual"] = np.array([st["final_residual"]])
            res[p + "step_max_disp"] = st["step_max_disp"]
        for where, pos in (("x", sc.x), ("y", sc.y)):
            P = O.search(sc, pos, 4e-3)
            srch[f"{tag}/{where}/keys"] = P.keys
            srch[f"{tag}/{where}/dist"] = P.dist
    np.savez_compressed(os.path.join(OUT, "resolve_fixtures.npz"), **res)
    np.savez_compressed(os.path.join(OUT, "search_fixtures.npz"), **srch)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
