"""RunConfig(profile=True): the five phases as separate timed kernels
(reference engine.py:489-500; acceptance C8 asserts every phase time is
> 0, test_acceptance.py:238-257).  The profile run is the same arithmetic
as the fused run and the per-phase API, so its state is bitwise the
reference's; its history rows carry each iteration's own phase times."""

import hashlib

import numpy as np
import pytest

from conftest import golden
import paper_1603_02526_b200 as fg

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def copy(st):
    return fg.AdmmState(*(np.array(getattr(st, k), copy=True) for k in "xmzun"),
                        iteration=st.iteration)


def test_profile_run_packing_bitwise_with_five_phase_times(gpu):
    gd = golden("pack100_seed0.npz")
    spec = fg.PackingSpec(100)
    g = fg.build_packing(spec)
    s = fg.packing_init(g, spec, seed=0)
    _sol, rep = fg.run(g, fg.RunConfig(max_iterations=10, profile=True), state=s)
    assert [sha(getattr(s, k)) for k in "xmzun"] == list(gd["sha_10"])
    assert all(rep.phase_seconds[p] > 0.0 for p in "xmzun")
    assert len(rep.history) == 10
    times = np.array([r[1:6] for r in rep.history])
    assert np.all(times > 0.0)
    # per-iteration rows, not one repeated mean
    assert len({tuple(t) for t in times}) > 1
    np.testing.assert_allclose(times.sum(axis=0),
                               [rep.phase_seconds[p] for p in "xmzun"], rtol=1e-12)
    np.testing.assert_allclose(np.array([r[-2:] for r in rep.history]), gd["hist_10"],
                               rtol=1e-12)
    csv = rep.metrics_csv().strip().split("\n")
    assert csv[0] == fg.METRICS_HEADER and len(csv) == 11


@pytest.mark.parametrize("seed", [None, 1])
def test_profile_run_svm_equals_fused_run(gpu, seed):
    """SVM chain graph: the fused run uses the SVM chain kernel, the
    profile run the unfused phases; both within 1e-9 of the reference
    golden, and the profile run bitwise the per-phase API."""
    gd = golden("svm200x32.npz")
    X, y = fg.gen_gaussian_arrays(200, 32, 4.0, seed=0)
    g = fg.build_svm(fg.SvmSpec.from_arrays(X, y))
    st = fg.init_state(g, seed=seed)
    tag = "zero" if seed is None else "seed1"
    s = copy(st)
    _sol, rep = fg.run(g, fg.RunConfig(max_iterations=10, profile=True), state=s)
    for k in "xmzun":
        ref = gd[f"{tag}_{k}_10"]
        assert np.max(np.abs(getattr(s, k) - ref)) <= 1e-9 * max(1.0, np.max(np.abs(ref)))
    s2 = copy(st)
    for _ in range(10):
        fg.iterate(g, s2)
    for k in "xmzun":
        np.testing.assert_array_equal(getattr(s, k), getattr(s2, k), err_msg=k)
    assert all(rep.phase_seconds[p] > 0.0 for p in "xmzun")


def test_profile_run_resumes_and_stops_like_fused(gpu):
    """Tolerance stop and resume: a profile run stops at the same
    iteration as the fused run, with the same state, and continues a
    state the fused run left (ping-pong slots shared)."""
    spec = fg.PackingSpec(10)
    g = fg.build_packing(spec)
    st = fg.packing_init(g, spec, seed=0)
    cfg = dict(max_iterations=5000, primal_tol=1e-6, dual_tol=1e-6)
    a, b = copy(st), copy(st)
    _s, ra = fg.run(g, fg.RunConfig(**cfg), state=a)
    _s, rb = fg.run(g, fg.RunConfig(**cfg, profile=True), state=b)
    assert ra.converged and rb.converged and ra.iterations == rb.iterations
    for k in "xmzun":
        np.testing.assert_array_equal(getattr(a, k), getattr(b, k), err_msg=k)
    c = copy(st)
    fg.run(g, fg.RunConfig(max_iterations=7), state=c)
    fg.run(g, fg.RunConfig(max_iterations=6, profile=True), state=c)
    fg.run(g, fg.RunConfig(max_iterations=5), state=c)
    d = copy(st)
    fg.run(g, fg.RunConfig(max_iterations=18), state=d)
    for k in "xmzun":
        np.testing.assert_array_equal(getattr(c, k), getattr(d, k), err_msg=k)
    assert c.iteration == 18


def test_profile_run_reports_failures_like_fused(gpu):
    b = fg.GraphBuilder()
    v = b.declare_variable(1)
    b.add_factor(fg.Quadratic([[1.0]], [1.0]), [v])
    b.add_factor(fg.NanTest("nan"), [v])
    g = b.freeze()
    with pytest.raises(RuntimeError, match=r"after x update at iteration 1: "
                                           r"edge 1 of factor 1 \(kind 'nan_test'\)"):
        fg.run(g, fg.RunConfig(max_iterations=3, profile=True))
    b = fg.GraphBuilder()
    w = b.declare_variable(1)
    v = b.declare_variable(1)
    b.add_factor(fg.Quadratic([[1.0]], [1.0]), [w])
    for _ in range(3):
        b.add_factor(fg.Quadratic([[1.7e308]], [1.0]), [v])
    g = b.freeze()
    with pytest.raises(RuntimeError,
                       match=r"non-finite value after z update at iteration 1: variable 1"):
        fg.run(g, fg.RunConfig(max_iterations=3, profile=True))
