"""GPU backend of the reference's benchmark command.

    python -m paper_1603_02526_b200.bench_cli pack --n 100,500 --iters 100
    python -m paper_1603_02526_b200.bench_cli mpc --k 10,100
    python -m paper_1603_02526_b200.bench_cli svm --n 1000 --workers 1,8

Same instances, flags, exit codes and CSV schema as ``fgadmm bench``
(reference cli.py:279-312, header :33-34): one row per (size, workers)
cell with the mean per-phase seconds of an iteration, the run's wall time,
time per iteration and the speedup against the 1-worker cell.  The phases
come from the device run in profile mode (RunConfig.profile: the five
phases as separate kernels, each bracketed by CUDA events every
iteration, as the reference's timers bracket them).  ``workers`` is
validated and, as in the
engine, does not change the device schedule.
"""

from __future__ import annotations

import argparse
import sys
from dataclasses import dataclass

import numpy as np

from . import engine
from .problems import (LinearSystem, MpcSpec, PackingSpec, SvmSpec, build_mpc, build_packing,
                       build_svm, gen_gaussian_data, packing_init, pendulum_linearization)

BENCH_HEADER = ("problem,size,workers,iters,"
                "t_x,t_m,t_z,t_u,t_n,total,time_per_iter,speedup")


@dataclass
class BenchResult:
    problem: str
    size: int
    workers: int
    iterations: int
    phase_means: dict
    total_seconds: float
    speedup: float

    @property
    def time_per_iteration(self):
        return sum(self.phase_means.values())

    def csv_row(self):
        cells = [self.problem, str(self.size), str(self.workers), str(self.iterations)]
        cells += [repr(float(self.phase_means[p])) for p in ("x", "m", "z", "u", "n")]
        cells += [repr(float(self.total_seconds)), repr(float(self.time_per_iteration)),
                  repr(float(self.speedup))]
        return ",".join(cells)


def bench_csv(results):
    return "\n".join([BENCH_HEADER] + [r.csv_row() for r in results]) + "\n"


class _Parser(argparse.ArgumentParser):
    """Usage failures exit with status 1 (reference cli.py:74-80)."""

    def error(self, message):
        self.print_usage(sys.stderr)
        sys.stderr.write(f"{self.prog}: error: {message}\n")
        raise SystemExit(1)


def _int_list(text):
    try:
        vals = [int(t) for t in text.split(",") if t.strip()]
    except ValueError as exc:
        raise argparse.ArgumentTypeError(f"not a comma-separated integer list: {text}") from exc
    if not vals or any(v < 1 for v in vals):
        raise argparse.ArgumentTypeError("sizes must be positive integers")
    return vals


def _instance(problem, size, seed):
    """The reference's bench instances (cli.py:266-276)."""
    if problem == "pack":
        spec = PackingSpec(size)
        graph = build_packing(spec)
        return graph, packing_init(graph, spec, seed=seed)
    if problem == "mpc":
        system = LinearSystem(*pendulum_linearization())
        return build_mpc(MpcSpec(size, system, np.array([0.0, 0.0, 0.1, 0.0]))), None
    points = gen_gaussian_data(size, 2, 4.0, seed=seed)
    return build_svm(SvmSpec(points)), None


def cmd_bench(args):
    sizes = args.k if args.problem == "mpc" else args.n
    if args.k is not None and args.problem != "mpc":
        raise RuntimeError("--k sizes only apply to the mpc problem")
    if args.n is not None and args.problem == "mpc":
        raise RuntimeError("mpc sizes are given with --k")
    if sizes is None:
        raise RuntimeError("no sizes given (use --n for pack/svm, --k for mpc)")
    results = []
    for size in sizes:
        cells = []
        for workers in args.workers or [1]:
            graph, state = _instance(args.problem, size, args.seed)
            cfg = engine.RunConfig(max_iterations=args.iters, workers=workers, profile=True)
            _sol, report = engine.run(graph, cfg, state=state)
            cells.append(BenchResult(args.problem, size, workers, report.iterations,
                                     report.mean_phase_seconds(), report.total_seconds, 1.0))
        base = next((c.time_per_iteration for c in cells if c.workers == 1),
                    cells[0].time_per_iteration)
        for c in cells:
            tpi = c.time_per_iteration
            c.speedup = base / tpi if tpi > 0 else float("nan")
        results.extend(cells)
    text = bench_csv(results)
    sys.stdout.write(text)
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(text)
    return 0


def build_parser():
    p = _Parser(prog="fgadmm-b200 bench",
                description="time fixed-iteration device runs over size sweeps")
    p.add_argument("problem", choices=("pack", "mpc", "svm"))
    p.add_argument("--n", type=_int_list, default=None)
    p.add_argument("--k", type=_int_list, default=None)
    p.add_argument("--workers", type=_int_list, default=None)
    p.add_argument("--iters", type=int, default=100)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--out")
    return p


def main(argv=None):
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as exc:
        return int(exc.code or 0)
    try:
        return cmd_bench(args)
    except KeyboardInterrupt:
        raise
    except Exception as exc:          # reference cli.py:326-328: exit code 2
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
