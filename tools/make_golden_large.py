"""Full-size goldens (CFG2 reef knot, CFG3 bow knot) from the REAL reference
build (oracle/_ref) and, for the device-coloring mode, from the C oracle.

The vectors are too large to commit, so tests/golden/large_digests.json holds
sha256 digests of their exact bytes plus the scalar stats:
  search/<scene>/<x|y>   sorted pair keys (u64) and distances (f64 bits) of
                         proximity_search at d_max = 4 mm
  resolve/<scene>/<mode> x_out bits, step_max_disp bits, steps, searches,
                         converged; mode "reference" = the reference build's
                         resolve (its own coloring), "device" = the C oracle's
                         statement of the device coloring
Scenes: the tightening targets of scenes.reef_knot / bow_knot at the bench's
squeeze (-0.2 mm: non-penetrating) and the penetrating frame tightening
(scenes.FRAME_DEFAULTS: +0.1 mm squeeze, 1.5 mm slide); delta
= 0.5 mm as in bench.py. The C oracle must agree with the reference bit for
bit in reference mode (asserted).

usage: python tools/make_golden_large.py [scene ...]   (~30 min on one core)
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import pyoracle as O  # noqa: E402
import pyref as R  # noqa: E402

from paper_2211_04045_b200 import scenes as S  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "large_digests.json")
DELTA = 5e-4


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def scenes():
    return {
        "reef": lambda: S.reef_knot(),
        "reef_pen": lambda: S.reef_knot(**S.FRAME_DEFAULTS),
        "bow": lambda: S.bow_knot(),
        "bow_pen": lambda: S.bow_knot(**S.FRAME_DEFAULTS),
    }


def main(names):
    out = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for name, make in scenes().items():
        if names and name not in names:
            continue
        sc = make()
        rm = R.RefMesh.from_scene(sc)
        assert np.array_equal(rm.edges(), sc.edges)
        rec = {"nv": int(sc.nv), "nt": int(len(sc.triangles)), "ne": int(len(sc.edges)),
               "x": sha(sc.x), "y": sha(sc.y)}
        for where, pos in (("x", sc.x), ("y", sc.y)):
            keys, dist, _ = R.search(rm, pos, 4e-3)
            rec[f"search_{where}"] = {"n": int(len(keys)), "keys": sha(keys), "dist": sha(dist)}
        t = time.time()
        xr, sr = R.resolve(rm, sc.x, sc.y, delta=DELTA)
        t_ref = time.time() - t
        xo, so = O.resolve(sc, delta=DELTA, coloring_mode="reference", trace=True)
        assert np.array_equal(xr.view(np.uint64), xo.view(np.uint64)), name
        assert np.array_equal(sr["step_max_disp"].view(np.uint64), so["step_max_disp"].view(np.uint64)), name
        rec["resolve_reference"] = {"x_out": sha(xr), "step_max_disp": sha(sr["step_max_disp"]),
                                    "steps": sr["steps"], "searches": sr["searches"],
                                    "converged": int(sr["converged"]), "ref_seconds": round(t_ref, 1),
                                    "trace": [[t["num_pairs"], t["num_contact_rows"], t["num_edge_rows"],
                                               t["num_colors"], t["num_active_pairs"]] for t in so["trace"]]}
        xd, sd = O.resolve(sc, delta=DELTA, coloring_mode="device", trace=True)
        rec["resolve_device"] = {"x_out": sha(xd), "step_max_disp": sha(sd["step_max_disp"]),
                                 "steps": sd["steps"], "searches": sd["searches"],
                                 "converged": int(sd["converged"]),
                                 "trace": [[t["num_pairs"], t["num_contact_rows"], t["num_edge_rows"],
                                            t["num_colors"], t["num_active_pairs"]] for t in sd["trace"]]}
        out[name] = rec
        json.dump(out, open(OUT, "w"), indent=1)
        print(name, "done", rec["resolve_reference"]["steps"], f"ref {t_ref:.0f}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
