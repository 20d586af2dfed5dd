"""``python -m paper_1604_08501_b200 {bench,check}`` — the GPU counterpart of
the reference CLI's ``bench`` and ``check`` subcommands (``lf/cli.py:77-117,
136-151``; SURVEY §2.1 lists a ``--device cuda`` bench mode as a follow-up).

* ``bench --nq N --ne N [--level L] [--seed S] [--check] [--emit FILE]
  [--report text|csv]`` — ``run_benchmark`` on the GPU: the reference's
  emitted level-L kernel (compiled for sm_100a) and this package's kernels,
  timed with CUDA events; exit 1 if the equivalence check exceeds 1e-5.
* ``check [--levels 1..8] [--nq 2,4,8] [--ne 1,2,5] [--seeds 1]`` — the
  equivalence suite (``full_check``) with every level's emitted kernel run
  on the GPU; levels the reference cannot emit are reported as SKIP.

Errors keep the reference's convention: ``LoopforgeError`` -> ``error: ...``
on stderr, exit code 1 (``lf/cli.py:158-162``). The reference's ``build``
subcommand (Fortran frontend + transform engine) is out of scope.
"""

from __future__ import annotations

import argparse
import sys

from .diagnostics import LoopforgeError
from .inputs import BenchmarkConfig


def _parse_int_list(text: str) -> list[int]:
    """``"1..8"`` or ``"2,3,4"`` (the reference's list syntax)."""
    out: list[int] = []
    for part in text.split(","):
        part = part.strip()
        if ".." in part:
            a, b = part.split("..")
            out.extend(range(int(a), int(b) + 1))
        elif part:
            out.append(int(part))
    return out


def _cmd_bench(args: argparse.Namespace) -> int:
    from .driver import BenchReport, run_benchmark
    cfg = BenchmarkConfig(nq=args.nq, ne=args.ne, level=args.level, seed=args.seed)
    report = run_benchmark(cfg, check=True if args.check else None)
    if args.emit:
        with open(args.emit, "w") as f:
            f.write(report.source)
    if args.report == "csv":
        print(BenchReport.csv_header())
        print(report.row_csv())
    else:
        print(report.row_text())
    if report.equivalence_error is not None and report.equivalence_error > 1e-5:
        print(f"error: equivalence failed ({report.equivalence_error:.3e} > 1e-5)",
              file=sys.stderr)
        return 1
    return 0


def _cmd_check(args: argparse.Namespace) -> int:
    from .driver import full_check
    failed = 0
    for cfg, err, ok in full_check(_parse_int_list(args.levels), _parse_int_list(args.nq),
                                   _parse_int_list(args.ne), _parse_int_list(args.seeds)):
        if err is None:
            print(f"level={cfg.level} Nq={cfg.nq} Ne={cfg.ne} seed={cfg.seed} "
                  f"SKIP (no emitted kernel for this level)")
            continue
        mark = "PASS" if ok else "FAIL"
        print(f"level={cfg.level} Nq={cfg.nq} Ne={cfg.ne} seed={cfg.seed} "
              f"rel_err={err:.3e} {mark}")
        failed += 0 if ok else 1
    if failed:
        print(f"error: {failed} configuration(s) failed", file=sys.stderr)
        return 1
    return 0


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(
        prog="paper_1604_08501_b200",
        description="the volume-term path of loopforge on B200 (sm_100a)")
    sub = parser.add_subparsers(dest="command", required=True)
    e = sub.add_parser("bench", help="time one corpus configuration on the GPU")
    e.add_argument("--nq", type=int, required=True)
    e.add_argument("--ne", type=int, required=True)
    e.add_argument("--level", type=int, default=8)
    e.add_argument("--seed", type=int, default=1)
    e.add_argument("--check", action="store_true",
                   help="force the equivalence check")
    e.add_argument("--emit", metavar="FILE", help="write the level's emitted source")
    e.add_argument("--report", choices=("text", "csv"), default="text")
    e.set_defaults(fn=_cmd_bench)
    c = sub.add_parser("check", help="equivalence suite on the GPU")
    c.add_argument("--levels", default="1..8")
    c.add_argument("--nq", default="2,4,8")
    c.add_argument("--ne", default="1,2,5")
    c.add_argument("--seeds", default="1")
    c.set_defaults(fn=_cmd_check)
    return parser


def main(argv: list[str] | None = None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.fn(args)
    except (LoopforgeError, ValueError) as err:
        print(f"error: {err}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
