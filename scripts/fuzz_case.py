"""Run one tests/test_gpu_fuzz.py case (its index as argv[1]) and print the plan and the error."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_1212_2245_b200 as md
from test_gpu_fuzz import _case, _oracle
for i in [int(a) for a in sys.argv[1:]]:
    psf, params, f, sigma, scen = _case(md, i)
    for dt in ("float64", "float32"):
        if dt == "float32" and not (sigma >= 5.0 and psf.kind is not md.PsfKind.GENERAL_2D):
            continue
        pipe = md.DeblurPipeline(f.shape, psf, params, scen, dtype=dt)
        print(i, dt, f.shape, scen, pipe.plan.describe, params, flush=True)
        out = pipe.run(f).values
        ref = _oracle(md, f, psf, params, scen)
        print("max|d|", float(np.abs(out - ref).max()), flush=True)
