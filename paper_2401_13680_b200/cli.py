"""Command line of the drop-in package: ``discover``, ``sweep``, ``label``, ``eval``.

Same subcommands, flags, JSON documents and exit codes as the reference CLI
(sniplab/cli.py:94-281): 0 = success, 1 = runtime
failure (ValueError / OSError / RuntimeError, message on stderr), 2 = usage
error.  Every heavy step goes through the package's GPU path; documents carry
``"schema": 1`` and do not depend on the number of GPUs/workers.

    python -m paper_2401_13680_b200 discover --input x.csv --m 120 --k 3
    python -m paper_2401_13680_b200 sweep --input x.csv --m-min 64 --m-max 512 --grid arith --step 32
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys


class UsageError(ValueError):
    """Invalid flag combination (exit code 2)."""


def _write_json(doc: dict, path: str | None) -> None:
    text = json.dumps(doc, indent=2) + "\n"
    if path is None:
        sys.stdout.write(text)
        return
    with open(path, "w") as fh:
        fh.write(text)


def _params(ns):
    from .mpdist import MPdistParams

    return MPdistParams(snippet_size=ns.m, window_size=ns.l, k=ns.mpdist_k)


def _exports(result, ns) -> None:
    from .snippets import export_curve_csv, export_profiles_csv

    if getattr(ns, "export_curve", None):
        export_curve_csv(result, ns.export_curve)
    if getattr(ns, "export_profiles", None):
        export_profiles_csv(result, ns.export_profiles)


def _validate(ns) -> None:
    """Cross-flag checks (the reference RunConfig rules, cli.py:57-74)."""
    if ns.command == "sweep":
        if ns.m_min > ns.m_max:
            raise UsageError(f"--m-min {ns.m_min} exceeds --m-max {ns.m_max}")
        if not 0.0 < ns.l_frac <= 1.0:
            raise UsageError(f"--l-frac must be in (0, 1], got {ns.l_frac}")
        if ns.workers is not None and ns.workers < 1:
            raise UsageError(f"--workers must be at least 1, got {ns.workers}")
    if getattr(ns, "k", 1) < 1:
        raise UsageError(f"--k must be at least 1, got {ns.k}")


def _columns(ns) -> list[int] | None:
    """--columns: multi-coordinate series (d > 1, Eq. 2) as the independent
    per-coordinate loop the reference prescribes (series.py:87-144):
    'all' or a comma list of zero-based CSV columns; None = single --column run."""
    spec = getattr(ns, "columns", None)
    if not spec:
        return None
    if spec == "all":
        import csv

        with open(ns.input, newline="") as fh:
            for row in csv.reader(fh):
                if row and any(cell.strip() for cell in row):
                    return list(range(len(row)))
        raise ValueError(f"series file {ns.input} has no rows")
    try:
        cols = [int(v) for v in spec.split(",")]
    except ValueError:
        raise UsageError(f"--columns must be 'all' or a comma list of column indices, got {spec!r}") from None
    if len(set(cols)) != len(cols) or min(cols) < 0:
        raise UsageError(f"--columns must list distinct non-negative indices, got {spec!r}")
    return cols


def _per_column(ns, run_one) -> int:
    """Run one subcommand per coordinate; JSON documents are collected as
    {"schema": 1, "coordinates": [{"column": c, ...}, ...]}, exports get a .c<col> suffix."""
    cols = _columns(ns)
    docs, extra = [], []
    out, out_snip = ns.output, getattr(ns, "output_snippets", None)
    exp = (getattr(ns, "export_curve", None), getattr(ns, "export_profiles", None))
    for c in cols:
        ns.column = c
        if exp[0]:
            ns.export_curve = f"{exp[0]}.c{c}"
        if exp[1]:
            ns.export_profiles = f"{exp[1]}.c{c}"
        d, e = run_one(ns)
        docs.append({"column": c, **d})
        if e is not None:
            extra.append({"column": c, **e})
    _write_json({"schema": 1, "coordinates": docs}, out)
    if out_snip:
        _write_json({"schema": 1, "coordinates": extra}, out_snip)
    return 0


def run_discover(ns) -> int:
    if _columns(ns) is not None:
        from .series import load_series
        from .snippets import select_snippets

        def one(ns):
            result = select_snippets(load_series(ns.input, column=ns.column), _params(ns), ns.k)
            _exports(result, ns)
            return result.to_dict(), None

        return _per_column(ns, one)
    return _run_discover_one(ns)


def _run_discover_one(ns) -> int:
    from .series import load_series
    from .snippets import select_snippets

    result = select_snippets(load_series(ns.input, column=ns.column), _params(ns), ns.k)
    _write_json(result.to_dict(), ns.output)
    _exports(result, ns)
    return 0


def _cost_model_from_log(path: str | None, n: int, enabled: bool):
    """Quadratic cost model from a training log with >= 3 distinct lengths (cli.py:109-117)."""
    from .scheduler import fit_cost_model, load_training_samples

    if not path or not enabled:
        return None
    try:
        sizes, seconds = load_training_samples(path, n)
    except FileNotFoundError:
        return None
    if len({float(s) for s in sizes}) < 3:
        return None
    return fit_cost_model(sizes, seconds, degree=2)


def run_sweep(ns) -> int:
    if _columns(ns) is not None:
        return _per_column(ns, _sweep_one)
    report, best = _sweep_one(ns, write=True)
    return 0


def _sweep_one(ns, write: bool = False):
    from .length_select import make_grid, select_length
    from .scheduler import TRAINING_LOG_ENV
    from .series import load_series

    series = load_series(ns.input, column=ns.column)
    grid = make_grid(ns.m_min, ns.m_max, rule=ns.grid, step=ns.step)
    log = ns.training_log or os.environ.get(TRAINING_LOG_ENV)
    frac = ns.l_frac

    def window_rule(m: int) -> int:  # l = max(1, min(m, ceil(m * l_frac)))
        return max(1, min(m, math.ceil(m * frac)))

    report, results = select_length(series, grid, ns.k, window_rule=window_rule, workers=ns.workers,
                                    cost_model=_cost_model_from_log(log, series.n, not ns.no_log),
                                    training_log=False if ns.no_log else log)
    best = results[report.m_best]
    _exports(best, ns)
    if write:
        _write_json(report.to_dict(), ns.output)
        if ns.output_snippets:
            _write_json(best.to_dict(), ns.output_snippets)
    return report.to_dict(), best.to_dict()


def run_label(ns) -> int:
    from .labeling import label_series, write_labels
    from .series import load_series
    from .snippets import select_snippets

    cols = _columns(ns)
    if cols is not None:  # one label column per coordinate
        import numpy as np

        lab = []
        for c in cols:
            ns.column = c
            lab.append(label_series(select_snippets(load_series(ns.input, column=c), _params(ns), ns.k)).labels)
        text = "".join(",".join(str(int(v)) for v in row) + "\n" for row in np.column_stack(lab))
        if ns.output is not None:
            with open(ns.output, "w") as fh:
                fh.write(text)
        else:
            sys.stdout.write(text)
        return 0

    labels = label_series(select_snippets(load_series(ns.input, column=ns.column), _params(ns), ns.k))
    if ns.output is not None:
        write_labels(labels, ns.output)
    else:
        sys.stdout.write("".join(f"{v}\n" for v in labels.labels))
    return 0


def run_eval(ns) -> int:
    from .labeling import evaluate, read_labels

    _write_json(evaluate(read_labels(ns.pred), read_labels(ns.truth)).to_dict(), ns.output)
    return 0


# (flags, kwargs) groups shared by the subcommands
_INPUT = [(("--input",), dict(required=True, help="series CSV, one value per line")),
          (("--column",), dict(type=int, default=0, help="CSV column to read")),
          (("--columns",), dict(default=None, help="multi-coordinate series: 'all' or a comma list of columns, "
                                                   "each processed independently (overrides --column)"))]
_FIXED_M = [(("--m",), dict(type=int, required=True, dest="m", help="snippet length")),
            (("--l",), dict(type=int, default=None, dest="l",
                            help="inner window length (default: half of --m, rounded up)")),
            (("--mpdist-k",), dict(type=int, default=None, help="MPdist order statistic (default: 5%% of 2m)"))]
_K = [(("--k",), dict(type=int, default=2, dest="k", help="number of snippets"))]
_OUT = [(("--output",), dict(default=None, help="write here instead of stdout"))]
_EXPORT = [(("--export-curve",), dict(default=None, help="representativeness curve CSV")),
           (("--export-profiles",), dict(default=None, help="snippet profiles CSV"))]
_SWEEP = [(("--m-min",), dict(type=int, required=True, help="smallest candidate length")),
          (("--m-max",), dict(type=int, required=True, help="largest candidate length")),
          (("--grid",), dict(choices=("pow2", "arith"), default="pow2")),
          (("--step",), dict(type=int, default=None, help="spacing for --grid arith")),
          (("--l-frac",), dict(type=float, default=0.5,
                               help="inner window length as a fraction of each candidate length")),
          (("--workers",), dict(type=int, default=None, help="GPU workers (default: SNIPLAB_WORKERS or 1)")),
          (("--training-log",), dict(default=None, help="JSON-lines timing log (default: SNIPLAB_TRAINING_LOG)")),
          (("--no-log",), dict(action="store_true", help="do not touch the training log")),
          (("--output-snippets",), dict(default=None, help="also write the winning length's snippet JSON here"))]
_EVAL = [(("--pred",), dict(required=True, help="predicted labels CSV")),
         (("--truth",), dict(required=True, help="ground-truth labels CSV"))]

COMMANDS = {
    "discover": (run_discover, "find snippets at a fixed length", _INPUT + _FIXED_M + _K + _OUT + _EXPORT),
    "sweep": (run_sweep, "pick the snippet length from a grid", _INPUT + _K + _OUT + _SWEEP + _EXPORT),
    "label": (run_label, "label every point with its nearest snippet", _INPUT + _FIXED_M + _K + _OUT),
    "eval": (run_eval, "score predicted labels against ground truth", _EVAL + _OUT),
}


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="paper_2401_13680_b200",
                                     description="Snippet discovery and labeling of time series on B200 GPUs.")
    sub = parser.add_subparsers(dest="command", required=True)
    for name, (_, help_text, flags) in COMMANDS.items():
        p = sub.add_parser(name, help=help_text)
        for names, kw in flags:
            p.add_argument(*names, **kw)
    return parser


def main(argv=None) -> int:
    try:
        ns = build_parser().parse_args(argv)
    except SystemExit as exc:  # argparse usage errors / --help
        return exc.code if isinstance(exc.code, int) else 2
    try:
        _validate(ns)
        return COMMANDS[ns.command][0](ns)
    except UsageError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    except (ValueError, OSError, RuntimeError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


def entry() -> None:
    sys.exit(main())
