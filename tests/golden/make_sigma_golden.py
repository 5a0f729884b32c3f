"""Writes sigma_from_seed.json: the shift σ of reading R3 ("i.i.d.
uniformly distributed in [0, Φ]") computed BY HAND from the PUBLISHED SplitMix64 outputs in
splitmix64.json (seed 1234567) — exact rational arithmetic, no oracle code:
    r_i = (z_i >> 11) · 2^-53,   σ_i = Φ · r_i  rounded once to the nearest double (ties to even),
which is what one IEEE-754 binary64 multiply of Φ by the exactly representable r_i gives.
Run: python tests/golden/make_sigma_golden.py"""
import json
import os
from fractions import Fraction

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
g = json.load(open(os.path.join(HERE, "splitmix64.json")))
outs = [int(z) for z in g["outputs"]]
cases = []
for phi32 in (1.0, 3.0, 0.7, 8.96):
    phi = float(np.float32(phi32))          # Φ of X = {0, phi32·1} in fp32, as the oracle reads it
    sig = [float(Fraction(phi) * Fraction(z >> 11, 1 << 53)) for z in outs]
    cases.append({"phi_f32": phi32, "phi": phi.hex(), "sigma": [s.hex() for s in sig]})
json.dump({"citation": "σ_i = Φ·((z_i >> 11)·2^-53) from the published SplitMix64 outputs of splitmix64.json "
                       "(reading R3 of PAPER.md:117); exact rational arithmetic, one rounding to binary64",
           "seed": g["seed"], "d": len(outs), "cases": cases},
          open(os.path.join(HERE, "sigma_from_seed.json"), "w"), indent=1)
