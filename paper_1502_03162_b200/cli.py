"""Command line for the render path: ``render``, ``render-all`` and ``bench``.

Mirrors the reference CLI's render and bench subcommands
(``cli.py:185-199,236-258``; parser ``cli.py:91-130``): same arguments,
exit codes (0 ok, 2 usage, 3 bad or missing data, 4 numerical failure) and
a ``run.json`` echoing the resolved configuration next to the output
(``cli.py:104-115``).  ``--backend`` accepts ``cuda`` (and ``compiled`` as an
alias); every convolution runs in the sm_100a kernels.  ``render-all`` is new:
one signal through every (ear, direction) of one model per ear in one fused
launch, written as ``[ears][directions][samples]`` float32 (``.npy`` or raw).

The preprocess / factorize / sparsify / reconstruct / metrics / tune-sigma
subcommands build the filters offline and are outside the render path.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

from . import __version__, engine, model_io
from .errors import DataError, NumericalError
from .types import Signal


def main(argv=None) -> int:
    parser = _parser()
    args = parser.parse_args(argv)
    if args.command is None:
        parser.print_help()
        return 2
    if args.command in ("render", "render-all") and not args.signal.lower().endswith(".wav") and args.rate is None:
        parser.error("headerless signal input needs --rate")
    try:
        _HANDLERS[args.command](args)
    except DataError as exc:
        print("data error: %s" % exc, file=sys.stderr)
        return 3
    except NumericalError as exc:
        print("numerical failure: %s" % exc, file=sys.stderr)
        return 4
    return 0


def _parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="toepnmf-b200",
                                     description="Render signals through factorized sparse HRIR models on a B200.")
    sub = parser.add_subparsers(dest="command")

    p = sub.add_parser("render", help="convolve a signal with one direction's response")
    p.add_argument("model", help="model JSON path")
    p.add_argument("signal", help="input signal (.wav, or headerless float32)")
    p.add_argument("--direction", type=int, required=True, help="direction index")
    p.add_argument("--out", required=True, help="output signal path (.wav or raw)")
    p.add_argument("--mode", choices=engine.MODES, default="sparse_direct", help="convolution mode")
    p.add_argument("--block-size", type=int, help="FFT block size override")
    p.add_argument("--backend", choices=("cuda", "compiled"), help="kernel backend (default cuda)")
    p.add_argument("--rate", type=float, help="sample rate for headerless input")

    p = sub.add_parser("render-all", help="render a signal through every direction of one model per ear")
    p.add_argument("models", nargs="+", help="model JSON path per ear (same directions and lengths)")
    p.add_argument("--signal", required=True, help="input signal (.wav, or headerless float32)")
    p.add_argument("--out", required=True, help="output: .npy, or raw float32 [ears][directions][samples]")
    p.add_argument("--rate", type=float, help="sample rate for headerless input")

    p = sub.add_parser("bench", help="time the convolution modes on random filters")
    p.add_argument("--signal-len", type=int, default=44100, help="benchmark signal length (default %(default)s)")
    p.add_argument("--nnze", default="1,2,5,10,25,50,100", help="comma-separated filter sizes (default %(default)s)")
    p.add_argument("--repeats", type=int, default=5, help="timed repeats per cell (default %(default)s)")
    p.add_argument("--block-size", type=int, help="FFT block size override")
    p.add_argument("--compare-backends", action="store_true", help="add a backend column")
    p.add_argument("--seed", type=int, default=0, help="filter/signal seed (default %(default)s)")
    p.add_argument("--out", required=True, help="output CSV path")
    return parser


def _require(path: str) -> str:
    if not os.path.exists(path):
        raise DataError("no such path: %s" % path)
    return path


def _write_run_json(primary_out: str, args, extra: dict | None = None) -> None:
    folder = primary_out if os.path.isdir(primary_out) else os.path.dirname(os.path.abspath(primary_out))
    doc = {"tool": "toepnmf-b200 %s" % __version__, "subcommand": args.command,
           "config": {k: v for k, v in vars(args).items() if k != "command"}}
    doc.update(extra or {})
    with open(os.path.join(folder, "run.json"), "w") as fh:
        json.dump(doc, fh, indent=2)
        fh.write("\n")


def _cmd_render(args) -> None:
    model = model_io.load_model(_require(args.model))
    sig = model_io.read_signal(_require(args.signal), sample_rate_hz=args.rate)
    out = engine.render(model, sig.samples, args.direction, mode=args.mode, block_size=args.block_size,
                        backend=args.backend)
    model_io.write_signal(Signal(samples=out, sample_rate_hz=sig.sample_rate_hz), args.out)
    _write_run_json(args.out, args)


def _cmd_render_all(args) -> None:
    for p in args.models:
        _require(p)
    sig = model_io.read_signal(_require(args.signal), sample_rate_hz=args.rate)
    br = model_io.load_renderer(args.models)
    out = br.render_all(sig.samples).cpu().numpy()
    if args.out.lower().endswith(".npy"):
        np.save(args.out, out)
    else:
        np.ascontiguousarray(out, dtype="<f4").tofile(args.out)
    _write_run_json(args.out, args, {"shape": list(out.shape), "sample_rate_hz": sig.sample_rate_hz})


def _cmd_bench(args) -> None:
    try:
        sizes = [int(v) for v in args.nnze.split(",") if v.strip()]
    except ValueError:
        raise DataError("could not parse --nnze %r" % args.nnze) from None
    backends = engine.available_backends() if args.compare_backends else None
    rows = engine.bench(args.signal_len, sizes, repeats=args.repeats, block_size=args.block_size,
                        backends=backends, seed=args.seed)
    engine.write_bench_csv(rows, args.out, include_backend=args.compare_backends)
    blocks = sorted({r.block_size for r in rows if r.block_size})
    _write_run_json(args.out, args, {"latency": {"fft_block_latency_samples": blocks,
                                                 "direct_latency_samples": 0,
                                                 "default_backend": engine.DEFAULT_BACKEND}})


_HANDLERS = {"render": _cmd_render, "render-all": _cmd_render_all, "bench": _cmd_bench}

if __name__ == "__main__":
    sys.exit(main())
