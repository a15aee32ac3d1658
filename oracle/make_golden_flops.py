"""Flop counts of the reference's ``qr_stacked_triangles`` for q-ary stacks
(householder.py:263-294 with its FlopCounter, counters.py:12-42), run on the
read-only reference: ``python oracle/make_golden_flops.py`` writes
``tests/golden/flops_stacked.json``."""

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.make_golden import OUT, load_reference  # noqa: E402

ref = load_reference()
out = {}
for n, q in [(8, 2), (8, 3), (16, 4), (32, 2)]:
    rng = ref["core"].rng_for(100 + q)
    Rs = [np.triu(rng.standard_normal((n, n))) for _ in range(q)]
    c = ref["counters"].FlopCounter()
    ref["householder"].qr_stacked_triangles(Rs, counter=c)
    out[f"{n}x{q}"] = [int(c.flops), int(c.divs)]
with open(os.path.join(OUT, "flops_stacked.json"), "w") as fh:
    json.dump(out, fh, indent=1)
print(out)
