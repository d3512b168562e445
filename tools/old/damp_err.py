import os, sys, numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2001_09632_b200 as p
from paper_2001_09632_b200 import _lib
z = np.load(os.path.join(ROOT, "tests/golden/family_cases.npz"))
ms = p.MeasurementSet(64, 64, 16, p.Algorithm.BBV, 1, 4, 0.0, z["counts"], z["coeffs"].astype(np.float32))
sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_recon_family import FAMILY, cfg_of
for name, *rest in FAMILY:
    res = p.reconstruct(ms, cfg_of(p, *rest), reference=z["img"])
    print(name, os.environ.get("ABCS_LIB", "new"), np.max(np.abs(res.image - z[f"{name}_x"])))
