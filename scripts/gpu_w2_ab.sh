# A/B of the 2W fold (robust weights stored doubled) against variants/libmdcuda_head.so
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/pytest_gpu.log
grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head
python - <<'PY'
import ctypes, os, torch, numpy as np
import paper_1212_2245_b200 as md
# bitwise comparison against the committed library on the c1 workload, f32 and f64
g = md.make_test_image(256, 256); psf = md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 15)
f = md.quantize(md.add_gaussian_noise(md.synth_blur(g, psf), 5.0, seed=5)).values
for dt in ("float32", "float64"):
    out = md.DeblurPipeline(f.shape, psf, md.DeconvParams(), dtype=dt).run(md.Image(f)).values
    np.save(f"gpurun_out/w2_{dt}.npy", out)
PY
MD_LIB=variants/libmdcuda_head.so python - <<'PY'
import numpy as np
import paper_1212_2245_b200 as md
g = md.make_test_image(256, 256); psf = md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 15)
f = md.quantize(md.add_gaussian_noise(md.synth_blur(g, psf), 5.0, seed=5)).values
for dt in ("float32", "float64"):
    out = md.DeblurPipeline(f.shape, psf, md.DeconvParams(), dtype=dt).run(md.Image(f)).values
    print(dt, "bitwise equal to head:", bool(np.array_equal(out, np.load(f"gpurun_out/w2_{dt}.npy"))))
PY
for r in 1 2; do for t in head base; do
  if [ "$t" = base ]; then L=""; else L=variants/libmdcuda_$t.so; fi
  MD_LIB=$L timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --e2e-batch 64 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1 $t', round(d['value']), d['stage_ms_per_step'])"
  MD_LIB=$L timeout 300 python bench.py --dtype float64 --steps 10 --warmup 3 --no-cpu --e2e-batch 64 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('f64 $t', round(d['value']), d['stage_ms_per_step'])"
done; done
