"""Command line front end (the reference's cli.py:132-289 deblur / bench / testimage / snr
subcommands) over the B200 library: ``python -m paper_1212_2245_b200 deblur in.pgm out.pgm
--psf box:h:15``. Exit codes: 0 ok, 1 usage error, 2 runtime error (cli.py:272-285)."""

from __future__ import annotations

import argparse
import os
import sys
import tempfile

from . import core, deconv, synth
from .benchmark import bench_pipeline, report
from .pgm import read_pgm, write_pgm

_SCEN = {"box": deconv.Scenario.BOX_1D, "fourier1d": deconv.Scenario.FOURIER_1D,
         "fourier2d": deconv.Scenario.FOURIER_2D}
_CONV = {deconv.Scenario.BOX_1D: "box", deconv.Scenario.FOURIER_1D: "fourier",
         deconv.Scenario.FOURIER_2D: "fourier2d"}


class UsageError(Exception):
    pass


def parse_psf_spec(spec: str) -> core.Psf:
    """``box:AXIS:LENGTH`` | ``line:LENGTH:ANGLE`` | ``file:PATH`` (core.py:260-312 text format)."""
    kind, _, rest = spec.partition(":")
    try:
        if kind == "box":
            axis, length = rest.split(":")
            return core.Psf.uniform_box(core.BlurAxis.parse(axis), float(length))
        if kind == "line":
            length, angle = rest.split(":")
            return core.Psf.line(float(length), float(angle))
        if kind == "file":
            return core.load_psf(rest)
    except (ValueError, OSError) as exc:
        raise UsageError(f"bad PSF spec {spec!r}: {exc}") from None
    raise UsageError(f"bad PSF spec {spec!r} (box:AXIS:LENGTH, line:LENGTH:ANGLE or file:PATH)")


def _params(a) -> core.DeconvParams:
    try:
        return core.DeconvParams(a.k, a.alpha, a.iters, a.eps_data, a.eps_reg, a.floor)
    except ValueError as exc:
        raise UsageError(str(exc)) from None


def _write(img, path):
    """Atomic write (cli.py:69-79)."""
    d = os.path.dirname(os.path.abspath(path))
    fd, tmp = tempfile.mkstemp(dir=d, suffix=".pgm")
    os.close(fd)
    try:
        write_pgm(img, tmp)
        os.replace(tmp, path)
    finally:
        if os.path.exists(tmp):
            os.remove(tmp)


def _scenario(flag, psf):
    return deconv.default_scenario(psf) if flag == "auto" else _SCEN[flag]


def cmd_deblur(a) -> int:
    psf, params = parse_psf_spec(a.psf), _params(a)
    f = read_pgm(a.input)
    scen = _scenario(a.scenario, psf)
    times = None
    if a.method == "wiener":
        out = (deconv.wiener_2d(f, psf, params.wiener_k, dtype=a.dtype) if scen is deconv.Scenario.FOURIER_2D
               else deconv.wiener_1d(f, psf, params.wiener_k, dtype=a.dtype))
    elif a.method == "rl":
        out = deconv.rl_deblur(f, psf, params.iterations, _CONV[scen], params.floor, dtype=a.dtype)
    elif a.method == "rrrl":
        out = deconv.rrrl_deblur(f, psf, params, _CONV[scen], dtype=a.dtype)
    else:
        out, times = deconv.DeblurPipeline(f.shape, psf, params, scen, dtype=a.dtype).run_timed(f)
    _write(out, a.output)
    if a.time and times is not None:
        print(f"wiener: {times.wiener_ms:.3f} ms")
        for i, ms in enumerate(times.iteration_ms, 1):
            print(f"rrrl iteration {i}: {ms:.3f} ms")
        print(f"rrrl total: {times.rrrl_total_ms:.3f} ms")
        print(f"total: {times.total_ms:.3f} ms")
    return 0


def cmd_bench(a) -> int:
    psf, params = parse_psf_spec(a.psf), _params(a)
    f = read_pgm(a.input)
    st = bench_pipeline(f, psf, params, _scenario(a.scenario, psf), runs=a.runs, warmup=a.warmup,
                        split_first_iteration=a.split_first_iteration, dtype=a.dtype)
    sys.stdout.write(report(st, a.format))
    return 0


def cmd_blur(a) -> int:
    psf = parse_psf_spec(a.psf)
    out = synth.synth_blur(read_pgm(a.input), psf)
    if a.noise != "none":
        kind, _, val = a.noise.partition(":")
        if kind == "gauss":
            out = synth.quantize(synth.add_gaussian_noise(out, float(val), a.seed))
        elif kind == "impulse":
            out = synth.quantize(synth.add_impulse_noise(out, float(val), a.seed))
        else:
            raise UsageError(f"bad noise spec {a.noise!r}")
    _write(out, a.output)
    return 0


def cmd_snr(a) -> int:
    print(f"{synth.snr(read_pgm(a.restored), read_pgm(a.reference)):.4f}")
    return 0


def cmd_testimage(a) -> int:
    _write(synth.make_test_image(a.width, a.height, a.seed), a.output)
    return 0


def _param_flags(p):
    p.add_argument("--psf", required=True, help="box:AXIS:LENGTH, line:LENGTH:ANGLE or file:PATH")
    p.add_argument("--k", type=float, default=0.006)
    p.add_argument("--alpha", type=float, default=0.003)
    p.add_argument("--iters", type=int, default=5)
    p.add_argument("--eps-data", type=float, default=1.0, dest="eps_data")
    p.add_argument("--eps-reg", type=float, default=0.01, dest="eps_reg")
    p.add_argument("--floor", type=float, default=0.1)
    p.add_argument("--scenario", default="auto", choices=["auto", "box", "fourier1d", "fourier2d"])
    p.add_argument("--dtype", default="float64", choices=["float64", "float32"])
    # the reference's thread-engine width (cli.py:215); accepted for drop-in command lines -- the
    # device runs the whole frame whatever its value (results do not depend on it, as in the
    # reference, parallel.py:10-13)
    p.add_argument("--threads", type=int, default=1, help="accepted for compatibility; the GPU runs the frame")


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_1212_2245_b200",
                                 description="Wiener + RRRL deconvolution on the B200")
    sub = ap.add_subparsers(dest="command", required=True)
    p = sub.add_parser("deblur")
    p.add_argument("input")
    p.add_argument("output")
    p.add_argument("--method", default="wr3l", choices=["wiener", "rl", "rrrl", "wr3l"])
    _param_flags(p)
    p.add_argument("--time", action="store_true")
    p.set_defaults(func=cmd_deblur)
    p = sub.add_parser("bench")
    p.add_argument("input")
    _param_flags(p)
    p.add_argument("--runs", type=int, default=100)
    p.add_argument("--format", default="human", choices=["human", "csv"])
    p.add_argument("--warmup", action="store_true")
    p.add_argument("--split-first-iteration", action="store_true", dest="split_first_iteration")
    p.set_defaults(func=cmd_bench)
    p = sub.add_parser("blur")
    p.add_argument("input")
    p.add_argument("output")
    p.add_argument("--psf", required=True)
    p.add_argument("--noise", default="none")
    p.add_argument("--seed", type=int, default=0)
    p.set_defaults(func=cmd_blur)
    p = sub.add_parser("snr")
    p.add_argument("restored")
    p.add_argument("reference")
    p.set_defaults(func=cmd_snr)
    p = sub.add_parser("testimage")
    p.add_argument("output")
    p.add_argument("--width", type=int, default=256)
    p.add_argument("--height", type=int, default=256)
    p.add_argument("--seed", type=int, default=7)
    p.set_defaults(func=cmd_testimage)
    return ap


def main(argv=None) -> int:
    try:
        a = build_parser().parse_args(argv)
    except SystemExit as exc:
        return 0 if exc.code in (0, None) else 1
    try:
        return a.func(a)
    except UsageError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    except (OSError, ValueError, RuntimeError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
