import hashlib, sys, os, warnings
sys.path.insert(0, os.getcwd())
warnings.simplefilter("ignore")
import numpy as np
from paper_1907_08560_b200 import ghsvd, inputs
P = inputs.known_hyperbolic(21, 600, 256, 0.5)
h = hashlib.sha256()
for kw in ({}, {"ordering": "hier", "super_blocks": 4}):
    ctx = ghsvd.Context(600, 256, variant="bo", **kw)
    ctx.set_factors(P.F, P.J, P.G)
    st = ctx.sweep()
    lam, sf, sg, Z = ctx.extract()
    ctx.close()
    h.update(lam.tobytes()); h.update(Z.tobytes()); h.update(str(st["sweeps"]).encode())
print("solve hash", h.hexdigest()[:16])
