"""Record the REAL reference's own acceptance outcomes (oracle/_ref/acceptance_groups,
the reference's tests/acceptance.cpp on the reference core) for the fast criterion
groups into tests/golden/reference_acceptance.json (the lines, verbatim)."""
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GROUPS = ["1_2_6", "3", "4", "10", "11"]
out = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "acceptance_groups")] + GROUPS, capture_output=True,
                     text=True).stdout
lines = [l for l in out.splitlines() if l.startswith("[")]
json.dump({"groups": GROUPS, "lines": lines}, open(os.path.join(ROOT, "tests", "golden", "reference_acceptance.json"), "w"),
          indent=1)
print("\n".join(lines))
