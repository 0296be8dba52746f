"""Command line of the device solver: ``python -m paper_2409_14222_b200
{run,sweep,stopping} ...`` with the subcommands, flags, TOML grid format and
CSV output of the reference's ``stokes-mg`` front end (``cli.py:22-91``).

    python -m paper_2409_14222_b200 run --case bdm --k 3 --levels 3 --out run.csv
    python -m paper_2409_14222_b200 sweep --config grid.toml --out sweep.csv
    python -m paper_2409_14222_b200 stopping --case th-quad --k 2 --max-levels 3 --out s.csv
"""

from __future__ import annotations

import argparse
import dataclasses
import sys
import tomllib

from . import experiments as E

_CHOICES = {"case": ["th-tri", "th-quad", "bdm", "rt"], "weighting": ["invmult", "unit"],
            "cheby": ["degree", "repeat"]}


def _parser() -> argparse.ArgumentParser:
    top = argparse.ArgumentParser(
        prog="python -m paper_2409_14222_b200",
        description="B200 multigrid-preconditioned solvers for the enclosed-flow benchmark on "
                    "the unit square")
    sub = top.add_subparsers(dest="command", required=True)

    run = sub.add_parser("run", help="solve one configuration")
    for f in dataclasses.fields(E.RunSpec):               # one flag per RunSpec field
        required = f.default is dataclasses.MISSING
        kind = {"int": int, "float": float, "float | None": float}.get(str(f.type), str)
        run.add_argument("--" + f.name.replace("_", "-"), type=kind, required=required,
                         default=None if required else f.default, choices=_CHOICES.get(f.name))
    run.add_argument("--out", required=True)

    grid = sub.add_parser("sweep", help="run a grid of configurations")
    grid.add_argument("--config", required=True, help="TOML table; k / nu / levels may be lists")
    grid.add_argument("--out", required=True)

    stop = sub.add_parser("stopping", help="find the loosest adequate tolerance")
    stop.add_argument("--case", required=True, choices=["th-quad", "bdm"])
    stop.add_argument("--k", type=int, required=True)
    stop.add_argument("--max-levels", type=int, required=True)
    stop.add_argument("--nu", type=int, default=1)
    stop.add_argument("--seed", type=int, default=0)
    stop.add_argument("--out", required=True)
    return top


def main(argv=None) -> int:
    args = _parser().parse_args(argv)
    if args.command == "run":
        spec = E.RunSpec(**{f.name: getattr(args, f.name) for f in dataclasses.fields(E.RunSpec)})
        row = E.run_case(spec).csv_row()
        with open(args.out, "w") as fh:
            fh.write(f"{E.CSV_COLUMNS}\n{row}\n")
        print(row)
        return 0
    with open(args.out, "w") as fh:
        if args.command == "sweep":
            with open(args.config, "rb") as cfg:
                rows = E.sweep(E.expand_grid(tomllib.load(cfg)), fh)
        else:
            rows = E.stopping_study(args.case, args.k, args.max_levels, nu=args.nu,
                                    seed=args.seed, out=fh)
    print(f"wrote {len(rows)} rows to {args.out}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
