"""``python -m paper_2605_29284_b200 <command> ...``: the reference CLI's commands on the GPU path.

Contract kept from the reference (cli.py): commands ``predict``, ``simulate``, ``bench-time``
(and ``bench-error`` / ``bench-converge``, outside this build's scope: exit 1); their flags;
the RKGRID1 output (interior grid, header extras sigma2 / alpha / nu / tau2 / covariates /
method / L [/ draws / seed / rng], fields ``prediction`` or ``mean`` / ``se`` [/ ``drawNNNN``]);
``RAPIDKRIG_SEED`` overriding ``--seed``; exit status 0 success, 1 usage or domain error,
2 numeric error.

Structure: every command is a ``Command`` subclass declaring its options as data and
implementing ``run``; ``cli_main`` builds the parser from those declarations and maps the
library's exception classes to exit codes through one table.
"""

from __future__ import annotations

import argparse
import csv
import os
import sys

from .covariance import CovarianceModel
from .errors import DomainError, NumericError, RapidKrigError
from .exact import fit, predict_exact
from .gridding import build_padded_grid
from .io import build_covariates, load_observations, parse_formula, write_grid_output
from .rapid import build_setup, predict_rapid
from .simulate import RNG_ALGORITHM, generate_ensemble
from .studies import run_timing

__all__ = ["cli_main", "main"]


class UsageError(DomainError):
    """Bad command line (exit 1, usage printed)."""


# ------------------------------------------------------------------ value parsers
def grid_spec(text: str):
    parts = text.lower().split("x")
    if len(parts) != 2 or not all(p.strip().isdigit() for p in parts):
        raise DomainError(f"bad grid spec {text!r}; expected e.g. 128x256")
    return int(parts[0]), int(parts[1])


def domain_spec(text: str):
    vals = text.split(",")
    if len(vals) != 4:
        raise DomainError(f"bad domain spec {text!r}; expected x0,x1,y0,y1")
    return tuple(map(float, vals))


def int_list(text: str):
    return tuple(int(v) for v in text.split(",") if v.strip())


def env_seed(default: int) -> int:
    v = os.environ.get("RAPIDKRIG_SEED")
    return int(v) if v else default


# ------------------------------------------------------------------ commands
class Command:
    name = ""
    help = ""
    options: tuple = ()          # (flags, argparse keyword arguments)

    def run(self, args) -> int:
        raise NotImplementedError


MODEL_AND_GRID = (
    ("--obs", dict(required=True, help="delimited text with x, y, z columns")),
    ("--out", dict(required=True, help="output grid file (RKGRID1)")),
    ("--grid", dict(required=True, type=grid_spec, metavar="M1xM2")),
    ("--domain", dict(type=domain_spec, default=None, help="x0,x1,y0,y1 (default: data bbox)")),
    ("--method", dict(choices=("exact", "rapid"), default="rapid")),
    ("--L", dict(type=int, default=4, help="neighbour order of the rapid method")),
    ("--covariates", dict(default="1", help="fixed-effect formula over 1, x, y, x*y")),
    ("--sigma2", dict(type=float, required=True)),
    ("--alpha", dict(type=float, required=True, help="Matern scale (1 / range)")),
    ("--nu", dict(type=float, required=True)),
    ("--tau2", dict(type=float, default=0.0)),
)


class Problem:
    """Observations, model, padded grid, covariates at data and nodes, GPU fit."""

    def __init__(self, args):
        self.args = args
        self.table = load_observations(args.obs)
        x0, x1, y0, y1 = self.table.bbox
        print(f"{args.obs}: {len(self.table)} observations in [{x0:g}, {x1:g}] x [{y0:g}, {y1:g}]")
        self.model = CovarianceModel(args.sigma2, args.alpha, args.nu, args.tau2)
        self.terms = parse_formula(args.covariates)
        self.grid = build_padded_grid(args.domain or self.table.bbox, args.grid, max(args.L, 1), self.table.locs)
        self.nodes = self.grid.interior_nodes()
        locs = self.table.locs
        self.krig = fit(self.model, locs, self.table.z, build_covariates(self.terms, locs[:, 0], locs[:, 1]))
        self.xg = build_covariates(self.terms, self.nodes[:, 0], self.nodes[:, 1])

    def setup(self):
        return build_setup(self.model, self.grid, self.args.L, self.table.locs)

    def save(self, fields, **extras):
        m1, m2 = self.grid.interior_dims
        meta = dict(sigma2=self.model.sigma2, alpha=self.model.alpha, nu=self.model.nu, tau2=self.model.tau2,
                    covariates="+".join(self.terms))
        meta.update(extras)
        (gx, gy), (hx, hy) = self.grid.origin, self.grid.spacing
        write_grid_output(self.args.out, nx=m1, ny=m2, x0=gx, y0=gy, dx=hx, dy=hy, fields=fields, extra=meta)
        print(f"{self.args.out}: {len(fields)} field(s) on the {m1}x{m2} interior grid")


class Predict(Command):
    name, help, options = "predict", "fit and predict onto a grid", MODEL_AND_GRID

    def run(self, args):
        pb = Problem(args)
        if args.method == "exact":
            m1, m2 = pb.grid.interior_dims
            field_ = predict_exact(pb.krig, pb.nodes, pb.xg).reshape(m2, m1)
        else:
            field_ = predict_rapid(pb.setup(), pb.krig.c, pb.krig.beta_hat, pb.xg)
        pb.save({"prediction": field_}, method=args.method, L=args.L)
        return 0


class Simulate(Command):
    name, help = "simulate", "conditional-simulation ensemble"
    options = MODEL_AND_GRID + (
        ("--draws", dict(type=int, default=100)),
        ("--seed", dict(type=int, default=0)),
        ("--save-draws", dict(action="store_true")),
    )

    def run(self, args):
        seed = env_seed(args.seed)
        pb = Problem(args)
        ens = generate_ensemble(pb.krig, pb.setup(), args.draws, seed, pb.xg, keep_draws=args.save_draws)
        fields = {"mean": ens.mean_field, "se": ens.empirical_se}
        if args.save_draws:
            fields.update(("draw%04d" % j, d) for j, d in enumerate(ens.draws))
        pb.save(fields, method="rapid", L=args.L, draws=args.draws, seed=seed, rng=RNG_ALGORITHM)
        return 0


class BenchTime(Command):
    name, help = "bench-time", "timing comparison on the GPU path"
    options = (
        ("--out", dict(required=True)),
        ("--ns", dict(type=int_list, default=(200, 1500))),
        ("--grids", dict(default="60x60,100x100,140x140")),
        ("--methods", dict(default="exact,rapid-L4")),
        ("--reps", dict(type=int, default=3)),
        ("--timeout", dict(type=float, default=60.0)),
        ("--seed", dict(type=int, default=1)),
    )
    COLUMNS = ("method", "n", "grid", "setup_seconds", "predict_seconds", "reps", "censored")

    def run(self, args):
        rows = run_timing(ns=args.ns, grid_ladder=tuple(map(grid_spec, args.grids.split(","))),
                          methods=tuple(m.strip() for m in args.methods.split(",")), reps=args.reps,
                          timeout_seconds=args.timeout, seed=env_seed(args.seed))
        with open(args.out, "w", newline="", encoding="utf-8") as fh:
            out = csv.writer(fh)
            out.writerow(self.COLUMNS)
            for r in rows:
                out.writerow([r.method, r.n, "%dx%d" % r.grid, "%.6f" % r.setup_seconds, "%.6f" % r.predict_seconds,
                              r.reps, int(r.censored)])
        print(f"{args.out}: {len(rows)} timing rows")
        return 0


class OutOfScope(Command):
    options = (("rest", dict(nargs="*")),)

    def __init__(self, name):
        self.name, self.help = name, "study harness (not in this build)"

    def run(self, args):
        raise DomainError(f"'{self.name}' (studies.py) is not provided by this build")


COMMANDS = (Predict(), Simulate(), BenchTime(), OutOfScope("bench-error"), OutOfScope("bench-converge"))


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        raise UsageError(f"{message}\n\n{self.format_usage()}")


def build_parser():
    top = _Parser(prog="rapidkrig", description="B200 rapid Kriging: predict / simulate / timing")
    sub = top.add_subparsers(dest="command", required=True)
    for cmd in COMMANDS:
        p = sub.add_parser(cmd.name, help=cmd.help)
        for flags, kw in cmd.options:
            p.add_argument(flags, **kw)
        p.set_defaults(_cmd=cmd)
    return top


# exception class -> (exit status, message prefix); first match wins
EXIT_CODES = ((UsageError, 1, ""), (NumericError, 2, "numeric error: "), (DomainError, 1, "error: "),
              (RapidKrigError, 2, "error: "))


def cli_main(argv=None) -> int:
    try:
        args = build_parser().parse_args(argv)
        return args._cmd.run(args)
    except RapidKrigError as err:
        for cls, status, prefix in EXIT_CODES:
            if isinstance(err, cls):
                print(f"{prefix}{err}", file=sys.stderr)
                return status
        raise


main = cli_main
