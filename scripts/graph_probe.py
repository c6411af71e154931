"""Per-call latency of the c1 pipeline, direct md_run vs CUDA-graph replay, at small batches
(host call + launches + device time, synchronised per call) and device time at 4096 frames."""
import json
import time

import numpy as np
import torch

import paper_1212_2245_b200 as md

psf = md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 15.0)
res = {}
for batch in (1, 16, 4096):
    pipe = md.DeblurPipeline((64, 128), psf, md.DeconvParams(), md.Scenario.BOX_1D, dtype="float32")
    x = torch.rand((batch, 64, 128), device="cuda") * 200 + 20
    g = pipe.capture(batch)
    g.f.copy_(x)
    out = torch.empty_like(x)
    for mode in ("run", "graph"):
        call = (lambda: pipe.plan.run(x, out)) if mode == "run" else g.replay
        for _ in range(20):
            call()
        torch.cuda.synchronize()
        reps = 200 if batch < 4096 else 20
        lat = []
        for _ in range(reps):
            t = time.perf_counter()
            call()
            torch.cuda.synchronize()
            lat.append((time.perf_counter() - t) * 1e3)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            call()
        e1.record()
        torch.cuda.synchronize()
        res[f"{mode}_b{batch}"] = {"p50_ms": float(np.median(lat)), "p99_ms": float(np.percentile(lat, 99)),
                                   "back_to_back_ms": e0.elapsed_time(e1) / reps}
    torch.cuda.synchronize()
    assert torch.equal(pipe.plan.run(x), g.replay())
print(json.dumps(res, indent=1))
