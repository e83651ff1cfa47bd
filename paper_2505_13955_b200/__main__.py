"""Command line: the GPU counterpart of `tomofuse reconstruct` (cli.py:153-159).

    python -m paper_2505_13955_b200 reconstruct SPECIMEN.sino --out DIR
        [--pitch 12] [--i0 1e5] [--window 0 4e-4] [--filter ramlak] [--feather 32]

writes DIR/volume.vol (uint16, the reference's VOL layout).  Errors map to
the reference's prefixes and exit code 2 (cli.py:264-285).
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path


def _parser():
    ap = argparse.ArgumentParser(prog="python -m paper_2505_13955_b200")
    sub = ap.add_subparsers(dest="command", required=True)
    r = sub.add_parser("reconstruct", help="FBP a SINO file into a uint16 VOL on the GPU")
    r.add_argument("sino", type=Path)
    r.add_argument("--out", type=Path, required=True)
    r.add_argument("--pitch", type=float, default=12.0, help="detector/voxel pitch in um (config.py:40,47)")
    r.add_argument("--i0", type=float, default=1e5)
    r.add_argument("--window", type=float, nargs=2, default=(0.0, 4e-4))
    r.add_argument("--filter", default="ramlak", choices=["ramlak", "shepplogan"])
    r.add_argument("--blur", type=float, default=0.0)
    r.add_argument("--feather", type=int, default=32)
    r.add_argument("--slab-rows", type=int, default=256)
    return ap


def cmd_reconstruct(args) -> int:
    from .fbp import FilterSpec, HuWindow
    from .formats import reconstruct_file

    spec = FilterSpec(kind=args.filter, blur_sigma=args.blur)
    win = HuWindow(*args.window)
    args.out.mkdir(parents=True, exist_ok=True)
    dst = args.out / "volume.vol"
    dims, dt = reconstruct_file(args.sino, dst, pixel_pitch=args.pitch, i0=args.i0, window=(win.lo, win.hi),
                                spec=spec, feather_band=args.feather, slab_rows=args.slab_rows)
    print(f"wrote {dst}; {dims.nx}x{dims.ny}x{dims.nz} in {dt:.3f} s (GPU pipeline)")
    return 0


def main(argv=None) -> int:
    from .formats import FormatError

    args = _parser().parse_args(argv)
    try:
        return {"reconstruct": cmd_reconstruct}[args.command](args)
    except Exception as exc:  # noqa: BLE001 - single exit point, like cli.py:274-285
        for klass, prefix in ((FormatError, "format error"), (FileNotFoundError, "io error"),
                              (ValueError, "input error")):
            if isinstance(exc, klass):
                print(f"{prefix}: {exc}", file=sys.stderr)
                return 2
        raise


if __name__ == "__main__":
    sys.exit(main())
