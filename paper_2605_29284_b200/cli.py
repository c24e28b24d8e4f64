"""``python -m paper_2605_29284_b200 predict|simulate ...`` on the GPU path (reference cli.py).

Same flags, output files and exit status as cli.py:60-263: 0 success, 1 domain / usage
error, 2 numeric error; ``RAPIDKRIG_SEED`` overrides ``--seed``.  ``predict`` fits on the GPU
and writes the ``prediction`` field by the rapid path (``--method rapid``, default) or exact
Kriging at every interior node (``--method exact``); ``simulate`` writes ``mean`` / ``se``
(and ``drawNNNN`` with ``--save-draws``) of a conditional-simulation ensemble;
``bench-time`` runs the timing study (studies.run_timing) and writes its CSV.  The error and
convergence studies (bench-error / bench-converge) are outside this build's scope and exit 1.
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


class _UsageError(DomainError):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        raise _UsageError(f"{message}\n\n{self.format_usage()}")


def _dims(text):
    try:
        a, b = text.lower().split("x")
        return int(a), int(b)
    except ValueError as err:
        raise DomainError(f"bad grid spec {text!r}; expected e.g. 128x256") from err


def _domain(text):
    parts = text.split(",")
    if len(parts) != 4:
        raise DomainError(f"bad domain spec {text!r}; expected x0,x1,y0,y1")
    return tuple(float(p) for p in parts)


def _parser():
    ap = _Parser(prog="rapidkrig", description="B200 rapid Kriging: predict / simulate")
    sub = ap.add_subparsers(dest="command", required=True)

    def common(p):
        p.add_argument("--obs", required=True, help="delimited text with x,y,z columns")
        p.add_argument("--out", required=True, help="output grid file (RKGRID1)")
        p.add_argument("--grid", required=True, type=_dims, metavar="M1xM2")
        p.add_argument("--domain", type=_domain, default=None, help="x0,x1,y0,y1 (default: data bbox)")
        p.add_argument("--method", choices=("exact", "rapid"), default="rapid")
        p.add_argument("--L", type=int, default=4, help="neighbour order of the rapid method")
        p.add_argument("--covariates", default="1", help="fixed-effect formula over 1,x,y,x*y")
        p.add_argument("--sigma2", type=float, required=True)
        p.add_argument("--alpha", type=float, required=True, help="Matern scale (1/range)")
        p.add_argument("--nu", type=float, required=True)
        p.add_argument("--tau2", type=float, default=0.0)

    common(sub.add_parser("predict", help="fit and predict onto a grid"))
    ps = sub.add_parser("simulate", help="conditional-simulation ensemble")
    common(ps)
    ps.add_argument("--draws", type=int, default=100)
    ps.add_argument("--seed", type=int, default=0)
    ps.add_argument("--save-draws", action="store_true")
    pt = sub.add_parser("bench-time", help="timing comparison (GPU path)")
    pt.add_argument("--out", required=True)
    pt.add_argument("--ns", type=lambda t: tuple(int(p) for p in t.split(",") if p.strip()), default=(200, 1500))
    pt.add_argument("--grids", default="60x60,100x100,140x140")
    pt.add_argument("--methods", default="exact,rapid-L4")
    pt.add_argument("--reps", type=int, default=3)
    pt.add_argument("--timeout", type=float, default=60.0)
    pt.add_argument("--seed", type=int, default=1)
    for name in ("bench-error", "bench-converge"):
        sub.add_parser(name, help="study harness (not in this build)").add_argument("rest", nargs="*")
    return ap


def _prepare(a):
    table = load_observations(a.obs)
    x0, x1, y0, y1 = table.bbox
    print(f"read {len(table)} observations from {a.obs}; bbox x [{x0:g}, {x1:g}] y [{y0:g}, {y1:g}]")
    domain = a.domain if a.domain is not None else table.bbox
    model = CovarianceModel(a.sigma2, a.alpha, a.nu, a.tau2)
    terms = parse_formula(a.covariates)
    grid = build_padded_grid(domain, a.grid, max(a.L, 1), table.locs)
    nodes = grid.interior_nodes()
    krig = fit(model, table.locs, table.z, build_covariates(terms, table.locs[:, 0], table.locs[:, 1]))
    return table, model, grid, nodes, build_covariates(terms, nodes[:, 0], nodes[:, 1]), krig, terms


def _write(a, grid, model, terms, fields, **meta):
    m1, m2 = grid.interior_dims
    extra = {"sigma2": model.sigma2, "alpha": model.alpha, "nu": model.nu, "tau2": model.tau2,
             "covariates": "+".join(terms), **meta}
    write_grid_output(a.out, nx=m1, ny=m2, x0=grid.origin[0], y0=grid.origin[1], dx=grid.spacing[0],
                      dy=grid.spacing[1], fields=fields, extra=extra)
    print(f"wrote {a.out} ({', '.join(fields)}; {m1}x{m2} grid)")


def _predict(a):
    table, model, grid, nodes, xg, krig, terms = _prepare(a)
    m1, m2 = grid.interior_dims
    if a.method == "exact":
        field = predict_exact(krig, nodes, xg).reshape(m2, m1)
    else:
        field = predict_rapid(build_setup(model, grid, a.L, table.locs), krig.c, krig.beta_hat, xg)
    _write(a, grid, model, terms, {"prediction": field}, method=a.method, L=a.L)
    return 0


def _simulate(a):
    env = os.environ.get("RAPIDKRIG_SEED")
    seed = int(env) if env else a.seed
    table, model, grid, nodes, xg, krig, terms = _prepare(a)
    ens = generate_ensemble(krig, build_setup(model, grid, a.L, table.locs), a.draws, seed, xg,
                            keep_draws=a.save_draws)
    fields = {"mean": ens.mean_field, "se": ens.empirical_se}
    if a.save_draws:
        fields.update({f"draw{j:04d}": ens.draws[j] for j in range(a.draws)})
    _write(a, grid, model, terms, fields, method="rapid", L=a.L, draws=a.draws, seed=seed, rng=RNG_ALGORITHM)
    return 0


def _bench_time(a):
    env = os.environ.get("RAPIDKRIG_SEED")
    rows = run_timing(ns=a.ns, grid_ladder=tuple(_dims(g) for g in a.grids.split(",")),
                      methods=tuple(m.strip() for m in a.methods.split(",")), reps=a.reps,
                      timeout_seconds=a.timeout, seed=int(env) if env else a.seed)
    with open(a.out, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh)
        w.writerow(("method", "n", "grid", "setup_seconds", "predict_seconds", "reps", "censored"))
        w.writerows((r.method, r.n, f"{r.grid[0]}x{r.grid[1]}", f"{r.setup_seconds:.6f}",
                     f"{r.predict_seconds:.6f}", r.reps, int(r.censored)) for r in rows)
    print(f"wrote {a.out} ({len(rows)} rows)")
    return 0


def _out_of_scope(a):
    raise DomainError(f"'{a.command}' (studies.py) is not provided by this build")


_COMMANDS = {"predict": _predict, "simulate": _simulate, "bench-time": _bench_time,
             "bench-error": _out_of_scope, "bench-converge": _out_of_scope}


def cli_main(argv=None) -> int:
    try:
        a = _parser().parse_args(argv)
        return _COMMANDS[a.command](a)
    except _UsageError as err:
        print(str(err), file=sys.stderr)
        return 1
    except NumericError as err:
        print(f"numeric error: {err}", file=sys.stderr)
        return 2
    except DomainError as err:
        print(f"error: {err}", file=sys.stderr)
        return 1
    except RapidKrigError as err:
        print(f"error: {err}", file=sys.stderr)
        return 2


main = cli_main
