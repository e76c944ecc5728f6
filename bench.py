"""Benchmark: ADMM edge-updates/sec of the B200 engine (and its roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload svm1m]
    python bench.py --impl reference ...      # CPU reference arm (fgadmm itself)

A step is one ADMM iteration (all five phases) over the whole graph.  The
default workload is BASELINE.json configs[1]: the soft-margin SVM chain on
1M synthetic Gaussian points x 32 dims (``build_svm``; zero init).  Other
workloads: pack5000 (configs[3]), mpc100k (configs[2]), pack100
(configs[0]).  One JSON line on stdout (rank 0).

value      = edges x K / device time of K iterations with the state resident
             in HBM (fused CUDA-graph loop, CUDA events on the engine stream;
             working set >> L2, so no flush is needed between steps).
e2e        = the same K iterations through the public ``run()`` call with
             host numpy state: state upload, K iterations, full-state
             download, measured by wall clock.
roofline   = dominant kernel's algorithmic bytes per launch / its average
             CUDA-event duration (``fg_profile_kernels``), against the
             measured HBM copy bandwidth in MEASURED_PEAKS.json.
cpu_baseline = the reference's own fgadmm.engine.run (installed under
             baseline/_ref) on a bounded sample of the same workload
             (the oracle port when it is not installed).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ADMM edge-updates/sec and HBM GB/s vs peak at 1/2/4/8 B200 vs CPU ref"
UNIT = "edge-updates/s"

WORKLOADS = {
    "svm1m": "soft-margin linear SVM chain, 1M points x 32 dims (configs[1])",
    "svm1m_rho2": "configs[1] with rho = 2 on every edge (SvmSpec(rho=2); adaptive-rho use case)",
    "svm1m_w": "configs[1] with rho = 1.5, alpha = 1.2 on every edge (non-power-of-two weights)",
    "pack5000": "circle packing N=5000 in the unit triangle (configs[3])",
    "mpc100k": "linear MPC, state 16, input 4, horizon 100k (configs[2])",
    "pack100": "circle packing N=100 in the unit triangle (configs[0])",
}


SVM_WEIGHTS = {"svm1m_rho2": (2.0, 1.0), "svm1m_w": (1.5, 1.2)}


def build_instance(name, scale=1.0):
    import paper_1603_02526_b200 as fg
    if name.startswith("svm"):
        n = int(1_000_000 * scale)
        X, y = fg.gen_gaussian_arrays(n, 32, 4.0, seed=0)
        rho, alpha = SVM_WEIGHTS.get(name, (1.0, 1.0))
        g = fg.build_svm(fg.SvmSpec.from_arrays(X, y, lam=1.0, rho=rho, alpha=alpha))
        return g, fg.init_state(g), {"points": n, "dim": 32, "init": "zeros",
                                     "rho": rho, "alpha": alpha}
    if name.startswith("pack"):
        n = int((5000 if name == "pack5000" else 100) * (scale if name == "pack5000" else 1))
        spec = fg.PackingSpec(n)
        g = fg.build_packing(spec)
        st = fg.packing_init(g, spec, seed=0)
        return g, st, {"disks": n, "init": "packing_init(seed=0)"}
    if name.startswith("mpc"):
        T = int(100_000 * scale)
        rng = np.random.default_rng(0)
        A = 0.05 * rng.standard_normal((16, 16))
        B = 0.1 * rng.standard_normal((16, 4))
        q0 = rng.standard_normal(16)
        g = fg.build_mpc(fg.MpcSpec(T, fg.LinearSystem(A, B), q0))
        return g, fg.init_state(g), {"horizon": T, "state_dim": 16, "input_dim": 4}
    raise SystemExit(f"unknown workload {name}")


# ---------------------------------------------------------------------------
# algorithmic bytes per kernel

def kernel_bytes(graph, plan):
    """Compulsory HBM bytes per launch of each kernel of one iteration, for
    the kernel forms the plan runs (unit-weight forms read no weights)."""
    dims = np.diff(np.asarray(graph.var_offsets))
    deg = np.bincount(graph.edge_var, minlength=len(dims))
    forms = plan.forms()
    out = {}
    for cls, sdims, fe, dp, _p, _s in plan.groups:
        B = len(fe)
        b = 0
        zcomp = 0
        wbytes = 0 if (cls.kind == "collision" and forms["collision_unit"]) else 8
        for j, d in enumerate(sdims):
            b += B * d * 16 + B * wbytes       # u read + x write, rho read
            zcomp += int(np.sum(dims[np.unique(graph.edge_var[fe + j])]))
        b += 8 * zcomp                         # z read once per component
        if dp.fparams is not None:
            b += dp.fparams.size * 8
        key = f"edge_{cls.kind}"
        out[key] = out.get(key, 0) + b
    small = deg <= 32
    chunk = 8192
    large = (~small) & (deg - 1 <= chunk)
    giant = (deg - 1) > chunk
    sel_by_key = [("var_small_deg4", deg <= 4), ("var_small_deg8", (deg > 4) & (deg <= 8)),
                  ("var_small_loop", small & (deg > 8))]
    for d in (1, 2, 3, 4):
        sel_by_key.append((f"var_large_d{d}", large & (dims == d)))
    sel_by_key.append(("var_large_comp", large & (dims > 4)))
    for key, sel in sel_by_key:
        if sel.any():
            P = int(np.sum(deg[sel] * dims[sel]))
            E = int(np.sum(deg[sel]))
            Z = int(np.sum(dims[sel]))
            unit = key.startswith("var_large_d") and forms["rows_unit"][int(key[-1])]
            out[key] = P * 24 + (0 if unit else E * 16) + Z * 24
    if giant.any():
        P = int(np.sum(deg[giant] * dims[giant]))
        E = int(np.sum(deg[giant]))
        out["var_giant_chunks"] = P * 16 + E * 8
        out["var_giant_update"] = P * 24 + E * 16
    out["reduce"] = 16 * (plan.info["small_components"] // 256 + 1
                          + plan.info["large_components"] + 64)
    if plan.info.get("fused_chain"):
        out["chain_svm"] = chain_bytes(graph, dims, deg, plan.chain_form() == "unit",
                                       forms.get("chain_uniform", False))
    if forms["chain"] == "mpc":
        # fused MPC chain: u read + write per payload double, z read +
        # write per component, the cost diagonal per component
        P, Z = graph.total_edge_payload, graph.z_dim
        out["chain_mpc"] = P * 16 + Z * 24
        # temporally blocked chain: the same compulsory bytes once per
        # launch of forms["mpc_block"] iterations (halo re-reads excluded)
        out["chain_mpc_block"] = P * 16 + Z * 24
    return out


def chain_bytes(graph, dims, deg, unit, uniform=False):
    """Compulsory bytes of one fused SVM-chain launch (csrc/fg_chain.cuh):
    per weight copy w_i (dim D, degree 3-4) u read+write and z read+write;
    per slack xi_i the same at dim 1, degree 2; per point the margin data
    (x_i, y_i), x.x, the norm and slack parameters, b's u read and x write.
    The weighted form also reads rho and alpha per edge of w_i and xi_i, one
    z weight per variable (w_i's is shared by its D components), b's rho
    and three per-point tables (norm factor, slack threshold, margin
    denominator); the unit-weight form reads none of them, and with uniform
    weights the weighted form reads the weights from a 4-double table
    (only the per-point tables are streamed).  Neighbours' equality edges
    are re-reads of the same arrays (L2), not counted."""
    n = int(np.sum(deg == 2))                  # xi's (b has degree n > 32)
    wsel = (deg >= 3) & (deg <= 4)
    P_w = int(np.sum(deg[wsel] * dims[wsel]))
    Z_w = int(np.sum(dims[wsel]))
    E_w = int(np.sum(deg[wsel]))
    V_w = int(np.sum(wsel))
    D = int(dims[wsel][0]) if wsel.any() else 0
    weights = not unit and not uniform
    w = P_w * 16 + Z_w * 16 + (E_w * 16 + V_w * 8 if weights else 0)
    xi = n * (2 * 16 + 16 + (2 * 16 + 8 if weights else 0))
    per_point = (D + 1) * 8 + 3 * 8 + 8 + 8 + (8 if weights else 0) + (0 if unit else 3 * 8)
    return w + xi + n * per_point


def survey_alg_bytes(graph):
    """B_alg = 40P + 32E + 24Z + 16V + B_par."""
    P, E, Z = graph.total_edge_payload, len(graph.edge_var), graph.z_dim
    V = len(graph.var_offsets) - 1
    bpar = 0
    for cls, dims, _f0, vars_, params in graph.blocks:
        if cls.kind == "svm_margin":
            bpar += vars_.shape[0] * 8 * (dims[0] + 1)
    return 40 * P + 32 * E + 24 * Z + 16 * V + bpar


# ---------------------------------------------------------------------------
# clocks

REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
           0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}


class ClockSampler:
    """SM clock and throttle reasons sampled every 5 ms through NVML while
    the timed region runs (the recipe's clocks line)."""

    def __init__(self, index=0, period=0.005):
        # NVML is initialised here, before the caller's warm-up: nvmlInit
        # takes milliseconds, and an idle GPU gap right before the timed
        # region lets the clocks drop.
        self.index = index
        self.period = period
        self.samples = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self._nv = None

    def __enter__(self):
        if self._nv is not None:
            self._stop.clear()
            self.samples = []
            self._t = threading.Thread(target=self._loop, daemon=True)
            self._t.start()
        return self

    def _loop(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.samples.append((float(sm), int(rs)))
            except Exception:
                break
            time.sleep(self.period)

    def __exit__(self, *exc):
        self._stop.set()
        if getattr(self, "_t", None) is not None:
            self._t.join(timeout=1.0)

    def summary(self):
        reasons = set()
        for _sm, mask in self.samples:
            for bit, name in REASONS.items():
                if mask & bit:
                    reasons.add(name)
        sm = [s for s, _m in self.samples]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml"}


# ---------------------------------------------------------------------------

def ncu_traffic(workload, kernel):
    """Per-launch DRAM bytes (read + write) of `kernel` from the committed
    ncu --set full capture summary (profiles/traffic.json, written by
    tools/traffic_json.py from the round's final_<workload>.ncu-rep)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            data = json.load(fh)
        return float(data[workload]["bytes_per_launch"][kernel])
    except (OSError, KeyError, ValueError):
        return None


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def reference_package():
    """The reference package ``fgadmm`` itself, installed unmodified under
    baseline/_ref (``pip install --no-index --target baseline/_ref``, see
    DESIGN.md section 7); None when it is not installed."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "fgadmm")):
        return None
    if path not in sys.path:
        sys.path.append(path)
    import fgadmm
    return fgadmm


def host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "cpu_count": os.cpu_count(),
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS")}


def reference_instance(ref, name, scale=1.0):
    """The workload built by the reference's OWN builders (problems.py),
    the same generators and specs as build_instance.  Packing starts from
    packing_init(seed=0): its arrays come from this package's replica,
    which is bit-identical to the reference's (tests/test_oracle.py) and
    O(N) faster; the graph layouts are identical (tests/test_documents.py)."""
    P = ref.problems
    if name.startswith("svm"):
        n = int(1_000_000 * scale)
        rho, alpha = SVM_WEIGHTS.get(name, (1.0, 1.0))
        g = P.build_svm(P.SvmSpec(P.gen_gaussian_data(n, 32, 4.0, seed=0), lam=1.0,
                                  rho=rho, alpha=alpha))
        return g, ref.init_state(g), {"points": n, "dim": 32, "init": "zeros"}
    if name.startswith("mpc"):
        T = int(100_000 * scale)
        rng = np.random.default_rng(0)
        A = 0.05 * rng.standard_normal((16, 16))
        B = 0.1 * rng.standard_normal((16, 4))
        q0 = rng.standard_normal(16)
        g = P.build_mpc(P.MpcSpec(T, ref.LinearSystem(A, B), q0))
        return g, ref.init_state(g), {"horizon": T, "state_dim": 16, "input_dim": 4}
    import paper_1603_02526_b200 as fg
    n = int((5000 if name == "pack5000" else 100) * (scale if name == "pack5000" else 1))
    g = P.build_packing(P.PackingSpec(n))
    og = fg.build_packing(fg.PackingSpec(n))
    st = fg.packing_init(og, fg.PackingSpec(n), seed=0)
    rs = ref.AdmmState(*(getattr(st, k) for k in "xmzun"))
    return g, rs, {"disks": n, "init": "packing_init(seed=0)"}


def _copy_ref_state(ref, st):
    return ref.AdmmState(*(np.array(getattr(st, k), copy=True) for k in "xmzun"))


def time_reference_run(ref, g, st, iterations, workers, record_every=None):
    """Seconds per iteration of fgadmm.engine.run itself (wall clock of the
    call; the report's total_seconds beside it)."""
    s = _copy_ref_state(ref, st)
    cfg = ref.RunConfig(max_iterations=iterations, workers=workers,
                        record_every=record_every or iterations)
    t0 = time.perf_counter()
    _sol, rep = ref.run(g, cfg, state=s)
    wall = time.perf_counter() - t0
    return wall / iterations, rep, s


def cpu_baseline(name, iters=None):
    """The reference's own fgadmm.engine.run (baseline/_ref; else the NumPy
    oracle port) on a bounded sample of the same workload: ~10-30 s of CPU
    work, the faster of 1 worker and one per host thread."""
    if name.startswith("svm"):
        scale, desc = 0.1, "SVM chain 100k x 32 (same generator)"
    elif name == "pack5000":
        scale, desc = 0.2, "packing N=1000 (same spec)"
    elif name.startswith("mpc"):
        scale, desc = 0.05, "MPC 16/4 horizon 5k (same generator)"
    else:
        scale, desc = 1.0, "packing N=100"
    ref = reference_package()
    if ref is not None:
        g, st, _info = reference_instance(ref, name, scale)
        E = len(g.edge_var)
        best = None
        for w in sorted({1, os.cpu_count() or 1}):
            time_reference_run(ref, g, st, 1, w)          # builds the lane plan
            tpi, _r, _s = time_reference_run(ref, g, st, 2, w)
            if best is None or tpi < best[0]:
                best = (tpi, w)
        n = iters or max(2, min(500, int(8.0 / max(best[0], 1e-6))))
        tpi, _r, _s = time_reference_run(ref, g, st, n, best[1])
        return {"value": E / tpi, "unit": UNIT, "cores": best[1], "kind": "reference",
                "sample": f"{desc}: fgadmm.engine.run (baseline/_ref), {n} iterations, "
                          f"workers={best[1]}, record_every={n}, {E} edges, "
                          f"{tpi * 1e3:.2f} ms/iter"}
    from oracle import fgadmm_oracle as O
    g, st, _info = build_instance(name, scale)
    o = O.Oracle(g)
    O.time_iterations(g, st, 1, oracle=o)             # warm caches
    t1, _ = O.time_iterations(g, st, 1, oracle=o)
    n = iters or max(2, min(200, int(8.0 / max(t1, 1e-6))))
    tpi, _ = O.time_iterations(g, st, n, oracle=o)
    E = len(g.edge_var)
    return {"value": E / tpi, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{desc}: {n} iterations, {E} edges, {tpi * 1e3:.2f} ms/iter"}


def reference_arm(args):
    """``--impl reference``: the reference's own CPU implementation,
    fgadmm.engine.run from baseline/_ref, on THIS workload at full size
    (pack5000 excepted: a 1/5-size sample, extrapolated per edge).  W
    warm-up iterations, then K timed iterations in one run() call
    (record_every = K), with the worker count that
    was faster in a short probe of 1 worker and one per host thread; the
    probe times and a record_every=1 (the reference default) run are
    reported beside it.  Without baseline/_ref the oracle port is timed."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    name = args.workload
    ref = reference_package()
    scale = 0.2 if name == "pack5000" else 1.0
    base = {"impl": "reference", "metric": METRIC, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic"}
    if ref is None:
        from oracle import fgadmm_oracle as O
        g, st, info = build_instance(name, scale)
        o = O.Oracle(g)
        s = O.State.copy_of(st)
        for _ in range(args.warmup):
            o.iterate(s)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            o.iterate(s)
        dt = time.perf_counter() - t0
        E = len(g.edge_var)
        value = E * args.steps / dt
        line = dict(base, value=value, ms_per_step=dt / args.steps * 1e3,
                    config={"workload": name, **info, "scale": scale,
                            "same_config": scale == 1.0},
                    cpu_baseline={"value": value, "unit": UNIT, "cores": 1, "kind": "port",
                                  "sample": f"oracle port, {E} edges per step"},
                    e2e={"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                         "d2h_bytes_per_step": 0},
                    host=host_info())
        print(json.dumps(line))
        return 0
    t_build = time.perf_counter()
    g, st, info = reference_instance(ref, name, scale)
    t_build = time.perf_counter() - t_build
    E = len(g.edge_var)
    ncpu = os.cpu_count() or 1
    probe = {}
    for w in sorted({1, ncpu}):
        time_reference_run(ref, g, st, 1, w)              # builds the lane plan
        tpi, _r, _s = time_reference_run(ref, g, st, 1, w)
        probe[w] = tpi
    best = min(probe, key=probe.get)
    s = _copy_ref_state(ref, st)
    if args.warmup:
        ref.run(g, ref.RunConfig(max_iterations=args.warmup, workers=best,
                                 record_every=args.warmup), state=s)
    t0 = time.perf_counter()
    _sol, rep = ref.run(g, ref.RunConfig(max_iterations=args.steps, workers=best,
                                         record_every=args.steps), state=s)
    dt = time.perf_counter() - t0
    value = E * args.steps / dt
    k1 = min(args.steps, 3)
    tpi1, _r1, _s1 = time_reference_run(ref, g, st, k1, best, record_every=1)
    line = dict(base, value=value, ms_per_step=dt / args.steps * 1e3,
                config={"workload": name, "desc": WORKLOADS[name], **info, "edges": E,
                        "scale": scale, "same_config": scale == 1.0,
                        "build_seconds": round(t_build, 1)},
                cpu_baseline={"value": value, "unit": UNIT, "cores": best,
                              "kind": "reference",
                              "sample": f"fgadmm.engine.run (unmodified reference, "
                                        f"baseline/_ref) on {E} edges, workers={best}, "
                                        f"record_every={args.steps}"
                                        + ("" if scale == 1.0 else
                                           f"; {scale:g}-scale sample, per-edge rate "
                                           f"extrapolated")},
                e2e={"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                     "d2h_bytes_per_step": 0},
                reference={"phase_seconds_per_iter": {k: v / args.steps for k, v in
                                                      rep.phase_seconds.items()},
                           "report_total_seconds": rep.total_seconds,
                           "probe_s_per_iter_by_workers": {str(k): v for k, v in probe.items()},
                           "workers": best,
                           "record_every_1": {"iterations": k1, "s_per_iter": tpi1,
                                              "value": E / tpi1}},
                host=host_info())
    print(json.dumps(line))
    return 0


def points_per_rank(args, world):
    """SVM points per rank of the weak-scaled run: --points-per-rank, else
    configs[4]'s 8M per GPU (64M at 8 GPUs) when the host can hold every
    local rank's graph and state (~8.5 KB per point, ~68 GB per rank at 8M
    points), else the largest whole million that fits (at least 1M)."""
    if args.points_per_rank:
        return args.points_per_rank
    # peak host bytes per point: the rank graph (~1.5 KB measured; the
    # per-payload zmap / rho_flat / alpha_flat are never built) plus the
    # page-locked five-array state (~5.2 KB) and the plan's transient
    # layout maps (~1.5 KB)
    target, per_point = 8_000_000, 8_500
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:                               # pragma: no cover
        return 1_000_000
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    fit = int(0.85 * avail / max(1, local_world) / per_point)
    return max(1_000_000, min(target, fit // 1_000_000 * 1_000_000))


def multi_gpu(args, fg, dist, rank, world, local):
    """N ranks over NCCL: the graph is partitioned by factors (cut variables
    all-gather their partial sums inside the iteration).

    SVM: weak scaling -- every rank holds n points (configs[4]: 8M per GPU,
    see points_per_rank) of a world x n-point chain and builds only its
    own part (partition.svm_rank_graph; cut set:
    the bias and one weight copy per rank boundary); value = all ranks'
    edges x K / max-rank time.  Packing / MPC: strong scaling of the one
    graph; each rank builds only its part from the spec
    (partition.packing_rank_graph / mpc_rank_graph, equal to
    Partition(...).local(rank))."""
    import torch
    from paper_1603_02526_b200.distributed import NcclRank
    from paper_1603_02526_b200.partition import svm_rank_graph
    t_build = time.perf_counter()
    weak = args.workload.startswith("svm")
    if weak:
        # every rank must hold the same number of points: the smallest
        # any rank's host memory allows
        nt = torch.tensor([points_per_rank(args, world)], device="cuda", dtype=torch.int64)
        dist.all_reduce(nt, op=dist.ReduceOp.MIN)
        n = int(nt.item())
        X, y = fg.gen_gaussian_arrays(n, 32, 4.0, seed=rank)
        lg = svm_rank_graph(X, y, rank, world, lam=1.0)
        nr = NcclRank(None, rank, world, device=local, local=lg, transport=args.transport)
        st = fg.init_state(lg)
        info = {"points": n * world, "points_per_rank": n, "dim": 32, "init": "zeros"}
        Et = torch.tensor([len(lg.edge_var)], device="cuda", dtype=torch.float64)
        dist.all_reduce(Et)
        E = int(Et.item())
    elif args.workload.startswith("mpc"):
        # strong scaling from the spec alone: each rank builds only its
        # part (partition.mpc_rank_graph; equal to Partition(...).local)
        from paper_1603_02526_b200.partition import mpc_rank_graph
        T = 100_000
        rng = np.random.default_rng(0)
        A = 0.05 * rng.standard_normal((16, 16))
        B = 0.1 * rng.standard_normal((16, 4))
        q0 = rng.standard_normal(16)
        spec = fg.MpcSpec(T, fg.LinearSystem(A, B), q0)
        lg = mpc_rank_graph(spec, rank, world)
        nr = NcclRank(None, rank, world, device=local, local=lg, transport=args.transport)
        st = fg.init_state(lg)
        info = {"horizon": T, "state_dim": 16, "input_dim": 4, "rank_graph": "mpc_rank_graph"}
        E = 3 * T + 2
    elif args.workload.startswith("pack"):
        # strong scaling from the spec alone (partition.packing_rank_graph)
        from paper_1603_02526_b200.partition import packing_rank_graph
        n = 5000 if args.workload == "pack5000" else 100
        spec = fg.PackingSpec(n)
        lg = packing_rank_graph(spec, rank, world)
        nr = NcclRank(None, rank, world, device=local, local=lg, transport=args.transport)
        st = fg.packing_init(lg, spec, seed=0)
        S = len(spec.planes)
        info = {"disks": n, "init": "packing_init(seed=0)", "rank_graph": "packing_rank_graph"}
        E = 4 * (n * (n - 1) // 2) + n + 2 * S * n
    else:
        g, st, info = build_instance(args.workload)
        nr = NcclRank(g, rank, world, device=local, transport=args.transport)
        E = len(g.edge_var)
    t_build = time.perf_counter() - t_build
    clk = ClockSampler(local)
    nr.upload(st)
    nr.run(args.warmup)
    nr.upload(st)
    torch.cuda.synchronize()
    dist.barrier()
    with clk:
        res, _hist = nr.run(args.steps)
    t = torch.tensor([res.ms_total], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = E * args.steps / (ms / 1e3)
    # end to end through the public per-rank API: scatter this rank's part
    # of the host state, run, download the rank's state (wall clock, max
    # over ranks)
    lg = nr.local
    pinned = True
    if nr.part is None:
        # rank graphs hold the rank's own state: page-locked like the 1-GPU
        # arm, downloaded back into the same arrays (as run() does); if the
        # host cannot pin that much, the pageable state is used (slower e2e)
        try:
            st_in = fg.pinned_state(lg, st)
            del st
        except Exception:                           # pragma: no cover
            st_in, pinned = st, False
        ls = [st_in.x, st_in.m, st_in.u, st_in.n]
        lz = st_in.z
    else:
        st_in, pinned = st, False
        ls = [np.empty(lg.total_edge_payload) for _ in range(4)]
        lz = np.empty(lg.z_dim)
    dist.barrier()
    t0 = time.perf_counter()
    nr.upload(st_in)
    nr.run(args.steps)
    nr.plan.download(x=ls[0], m=ls[1], z=lz, u=ls[2], n=ls[3])
    e2e_s = torch.tensor([time.perf_counter() - t0], device="cuda")
    dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    P_all = torch.tensor([lg.total_edge_payload, lg.z_dim], device="cuda", dtype=torch.float64)
    dist.all_reduce(P_all)
    P_tot, Z_tot = float(P_all[0].item()), float(P_all[1].item())
    e2e = {"value": E * args.steps / float(e2e_s.item()), "unit": UNIT,
           "h2d_bytes_per_step": int((Z_tot + 2 * P_tot) * 8 // args.steps),
           "d2h_bytes_per_step": int((4 * P_tot + Z_tot) * 8 // args.steps),
           "pinned": pinned,
           "note": "per rank: upload its part of z,u,n, run, download its x,m,z,u,n; "
                   "max over ranks of the wall clock"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak" if weak else "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload,
                   "desc": (f"soft-margin linear SVM chain, {info['points_per_rank'] / 1e6:g}M points "
                            f"per GPU x 32 dims, weak-scaled (configs[4]: 8M per GPU, 64M at 8)"
                            if weak else WORKLOADS[args.workload]), **info,
                   "edges": E, "parallelism": f"factor partition x{world} ({args.transport.upper()} all-gather "
                                              f"of {getattr(nr.local, 'ncut', 0)} cut components)",
                   "transport": args.transport,
                   "local_edges": len(nr.local.edge_var), "build_seconds": round(t_build, 2),
                   "host_max_rss_gb": round(__import__("resource").getrusage(
                       __import__("resource").RUSAGE_SELF).ru_maxrss / 2**20, 1)},
        "gpu_launches": int(res.launches), "clocks": clk.summary(),
        "converged": bool(res.converged),
        "e2e": e2e,
        "roofline": None, "cpu_baseline": None,
        "note": "roofline and the CPU baseline are reported by the one-GPU line",
        "chain_form": nr.plan.chain_form(),
    }
    if rank == 0:
        print(json.dumps(line))
    dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="svm1m", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--partition", action="store_true",
                    help="take the multi-GPU (NCCL partition) path even at one rank")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "p2p"],
                    help="multi-GPU cut/residual exchange: NCCL all-gather, or peer-memory "
                         "stores over NVLink with epoch flags (CUDA IPC)")
    ap.add_argument("--points-per-rank", type=int, default=None,
                    help="SVM points per rank of the weak-scaled multi-GPU run "
                         "(default configs[4]: 8M per GPU = 64M at 8 GPUs, fewer "
                         "when the host memory cannot hold all local ranks)")
    args = ap.parse_args()
    if args.impl == "reference":
        return reference_arm(args)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    os.environ["FGADMM_DEVICE"] = str(local)
    dist = None
    if world > 1 or args.partition:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")

    import paper_1603_02526_b200 as fg
    if world > 1 or args.partition:
        return multi_gpu(args, fg, dist, rank, world, local)
    t_build = time.perf_counter()
    g, st, info = build_instance(args.workload)
    plan = fg.device_plan(g)
    t_build = time.perf_counter() - t_build
    E = len(g.edge_var)

    # ---- device-resident timed region ----
    clk = ClockSampler(local)
    plan.sync(g)
    plan.upload(st.z, st.u, st.n)
    wres, _ = plan.run(args.warmup)                        # untimed warm-up
    # clock settle: an idle GPU ramps its clocks back up over milliseconds,
    # so latency-bound workloads (< 0.25 ms per iteration) keep warming
    # (untimed) until ~0.1 s of device work; bandwidth-bound ones are not
    # held at full power longer than the warm-up asks (power capping)
    warm_ms, settle = wres.ms_total, 0
    short = wres.ms_total / max(args.warmup, 1) < 0.25
    while short and warm_ms < 100.0 and settle < 100000:
        n = max(args.warmup, 20)
        wres, _ = plan.run(n)
        warm_ms += wres.ms_total
        settle += n
    if dist:
        dist.barrier()
    with clk:
        res, _hist = plan.run(args.steps, graph_chunk=16)
    ms = res.ms_total
    if dist:
        import torch
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = E * args.steps * world / (ms / 1e3)

    # ---- per-kernel profile (same arithmetic, events per launch) ----
    plan.upload(st.z, st.u, st.n)
    prof = plan.profile_kernels(max(3, min(args.steps, 20)))
    kb = kernel_bytes(g, plan)
    top = max(prof, key=lambda k: prof[k][0])
    base = top.split("#")[0]
    avg_ms = prof[top][0] / prof[top][1]
    peak, peak_kind = measured_peak()
    achieved = kb.get(base, 0) / (avg_ms / 1e3) / 1e9
    # a temporally blocked launch covers several iterations
    its_per_launch = plan.forms()["mpc_block"] if base == "chain_mpc_block" else 1
    iter_bytes = sum(kb.get(k.split("#")[0], 0) for k in prof) / its_per_launch
    iter_ms = sum(v[0] for v in prof.values()) / prof[top][1] / its_per_launch
    fp64 = None
    if base == "chain_mpc_block":
        # the dynamics products v = K nv: 2 cols^2 flops per factor per
        # iteration (halo recomputation not counted)
        T = info["horizon"]
        flops = its_per_launch * T * 2 * 36 * 36
        fp64 = {"flops_per_launch": flops, "TFLOPs": flops / (avg_ms / 1e3) / 1e12,
                "note": "the blocked chain reads its state once per launch; its "
                        "per-launch time is set by the fp64 dynamics products and "
                        "shared-memory traffic, not HBM",
                "limiter": "K nv on the fp64 tensor cores (mma.sync m8n8k4); the rest is "
                           "shared-memory traffic and issue; DRAM 11% "
                           "(profiles/r02_ncu_mpc100k.md)"}

    # ---- end to end through the public API (host state in, host state out) ----
    # three calls, each from the same initial state; the median is reported
    s = fg.pinned_state(g, st)                     # page-locked host arrays
    e2e_runs = []
    for _ in range(3):
        for k in ("z", "u", "n"):
            getattr(s, k)[...] = getattr(st, k)
        s.iteration = st.iteration
        t0 = time.perf_counter()
        fg.run(g, fg.RunConfig(max_iterations=args.steps), state=s)
        e2e_runs.append(time.perf_counter() - t0)
    e2e_s = float(np.median(e2e_runs))
    P, Z = g.total_edge_payload, g.z_dim
    h2d = (Z + 2 * P) * 8 + 2 * E * 8 * 0
    d2h = (4 * P + Z) * 8
    loop_s = ms / 1e3                              # device time of the same iterations
    xfer_s = e2e_s - loop_s
    e2e = {"value": E * args.steps * world / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps,
           "runs_s": [round(v, 4) for v in e2e_runs],
           "device_loop_s": round(loop_s, 5),
           "host_transfer_GBps": (round((h2d + d2h) / xfer_s / 1e9, 1)
                                  if xfer_s > 0.05 * e2e_s else None),
           "bound": "pcie",
           "note": f"one run() call of {args.steps} iterations on a pinned host "
                   f"AdmmState: upload z,u,n, download x,m,z,u,n (bytes amortized "
                   f"per step); wall clock, median of 3 calls.  Transfer-dominated: "
                   f"{(h2d + d2h) / 1e9:.2f} GB cross PCIe per call against "
                   f"{loop_s * 1e3:.1f} ms of device loop; host_transfer_GBps is "
                   f"the call's bytes over its non-loop time"}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0
    cpu = None if args.no_cpu_baseline or world > 1 else cpu_baseline(args.workload)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "desc": WORKLOADS[args.workload], **info,
                   "edges": E, "payload": g.total_edge_payload, "z_dim": g.z_dim,
                   "parallelism": "replicas" if world > 1 else "single",
                   "l2": "working set > L2 (no flush needed)",
                   "warmup_settle_steps": settle,
                   "build_seconds": round(t_build, 2)},
        "roofline": {"bound": "hbm", "kernel": top, "achieved": achieved, "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": ncu_traffic(args.workload, base),
                     "alg_bytes": kb.get(base, 0),
                     "iterations_per_launch": its_per_launch, "fp64": fp64,
                     "iteration": {"alg_bytes": iter_bytes,
                                   "survey_B_alg": survey_alg_bytes(g),
                                   "ms": iter_ms,
                                   "GBps": iter_bytes / (iter_ms / 1e3) / 1e9},
                     # EU/s against the two-pass roofline
                     # (peak x E / B_alg); above 1 when the fused schedules
                     # move fewer bytes than the two-pass minimum
                     "survey_roofline_EUps": peak * 1e9 * E / survey_alg_bytes(g) * world,
                     "value_over_survey_roofline":
                         value / (peak * 1e9 * E / survey_alg_bytes(g) * world)},
        "kernels": {k: {"ms_avg": v[0] / v[1], "alg_bytes": kb.get(k.split("#")[0], 0)}
                    for k, v in prof.items()},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(res.launches),
        "clocks": clk.summary(),
    }
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
