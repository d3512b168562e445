import os, sys, numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle")); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2001_09632_b200 as p
import oracle as o
from test_recon_family import cfg_of
z = np.load(os.path.join(ROOT, "tests/golden/family_cases.npz"))
ref = o.Reference()
ms = p.MeasurementSet(64, 64, 16, p.Algorithm.BBV, 1, 4, 0.0, z["counts"], z["coeffs"].astype(np.float32))
for it in (1, 2, 3, 4, 5):
    res = p.reconstruct(ms, cfg_of(p, 3, it, 1.0, 42, "dct_threshold", 25.0, 2.0), reference=z["img"])
    wx, wt = ref.reconstruct(4, 4, 16, z["counts"], z["coeffs"].astype(np.float32).astype(np.float64), 3, it, 2.0, 1.0, 42, 0, 2.7, 8, 25.0, ref=z["img"])
    d = np.abs(res.image - wx)
    print(os.environ.get("ABCS_LIB", "new"), it, f"max {d.max():.2e} mean {d.mean():.2e} argmax {np.unravel_index(d.argmax(), d.shape)} sigma {res.trace[-1].sigma:.6f} vs {wt[-1,2]:.6f}")
