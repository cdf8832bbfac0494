"""The reference's OWN acceptance suite (proj/tests/acceptance.cpp, unmodified)
compiled against this repository's drop-in headers (include/twoway, with the
Eigen-subset shim standing in for Eigen) and linked to libtwoway_b200.so in
place of the reference core (oracle/_ref/b200/acceptance_groups, built by
oracle/Makefile.ref; the reference's dynamics / normal-flow / testkit sources
recompiled unchanged on top). Every resolve, proximity search, linearize,
assemble_lcp, pgs_sweeps and constraint_value_at it calls runs on the B200.

With TWOWAY_COLORING=reference (the bit-exact Gauss-Seidel order) every
criterion line must equal the real reference's own line
(tests/golden/reference_acceptance.json, from oracle/_ref/acceptance_groups:
the same suite on the reference core) character for character -- including
the two criteria the reference itself fails (#4: constraint FD error 6.04e-04
> 1e-4; #11: stretch 1.345 > 1.15). With the default device coloring the
pass/fail outcomes must match except #11, where the device order lands
closer to the threshold."""
import json
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "b200", "acceptance_groups")
GOLD = os.path.join(ROOT, "tests", "golden", "reference_acceptance.json")


def _run(env_extra):
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/b200/acceptance_groups not built")
    gold = json.load(open(GOLD))
    env = dict(os.environ, **env_extra)
    out = subprocess.run([EXE] + gold["groups"], capture_output=True, text=True, env=env, timeout=1200).stdout
    return gold, [l for l in out.splitlines() if l.startswith("[")]


def _outcomes(lines):
    return {int(m.group(2)): m.group(1) for m in (re.match(r"\[(\w+)\] criterion\s+(\d+)", l) for l in lines) if m}


def test_acceptance_reference_coloring_is_the_references():
    gold, lines = _run({"TWOWAY_COLORING": "reference"})
    assert lines == gold["lines"]


def test_acceptance_device_coloring_outcomes():
    gold, lines = _run({})
    ours, ref = _outcomes(lines), _outcomes(gold["lines"])
    assert set(ours) == set(ref)
    for k in ref:
        if k != 11:
            assert ours[k] == ref[k], (k, lines)
    assert ours[1] == ours[2] == ours[3] == ours[6] == ours[10] == "PASS"
