"""Graph documents (reference graph.py:265-340) and the
drop-in boundary for the reference's own ``FactorGraph`` objects.

* documents WRITTEN BY THE REFERENCE (tests/golden/doc_*.json.gz, made by
  tests/golden/make_golden.py) deserialize into graphs with the
  reference's flat layout and serialize back byte for byte;
* the six rejection cases of the reference's test_graph.py:134-196;
* where the reference is importable: a reference ``fgadmm.FactorGraph``
  yields the same kind groups (``_group_specs``: kinds, slot dims, first
  edges, packed device parameters) and layout arrays as this package's
  graph of the same problem -- what ``engine.run`` reads when it is handed
  a reference graph (engine.py:_group_specs else-branch).
"""

import gzip
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden, import_reference
import paper_1603_02526_b200 as fg
from paper_1603_02526_b200.engine import _group_specs

DOCS = ("pack30", "svm60x4", "mpc4x2")


def read_doc(tag):
    with gzip.open(os.path.join(GOLDEN, f"doc_{tag}.json.gz"), "rt") as fh:
        return fh.read()


@pytest.mark.parametrize("tag", DOCS)
def test_reference_document_round_trip_byte_identical(tag):
    gd = golden("documents.npz")
    doc = read_doc(tag)
    assert hashlib.sha256(doc.encode()).hexdigest() == str(gd[f"{tag}_doc_sha"])
    g = fg.deserialize(doc)
    assert fg.serialize(g) == doc
    for key in ("zmap", "z_weights", "rho_flat", "alpha_flat"):
        np.testing.assert_array_equal(getattr(g, key), gd[f"{tag}_{key}"], err_msg=key)


def two_quadratic_graph():
    b = fg.GraphBuilder()
    w = b.declare_variable(1)
    b.add_factor(fg.Quadratic([[1.0]], [1.0]), [w])
    b.add_factor(fg.Quadratic([[3.0]], [1.0]), [w])
    return b.freeze()


def test_wall_radius_round_trip():
    """test_graph.py:134-150."""
    b = fg.GraphBuilder()
    c = b.declare_variable(2)
    r = b.declare_variable(1)
    plane = fg.HalfPlane((0.6, 0.8), (0.25, -1.5))
    b.add_factor(fg.Wall(plane), [c, r], rho=[1.25, 2.5], alpha=0.9)
    b.add_factor(fg.Radius(0.5), [r], rho=5.0)
    g = b.freeze()
    doc = fg.serialize(g)
    g2 = fg.deserialize(doc)
    assert fg.serialize(g2) == doc
    assert g2.counts() == g.counts()
    np.testing.assert_array_equal(g2.rho_flat, g.rho_flat)
    np.testing.assert_array_equal(g2.alpha_flat, g.alpha_flat)
    assert [f.operator.kind for f in g2.factors] == ["wall", "radius"]


def test_document_shape():
    doc = json.loads(fg.serialize(two_quadratic_graph()))
    assert doc["version"] == fg.DOCUMENT_VERSION
    assert doc["variables"] == [{"id": 0, "dim": 1}]
    assert doc["factors"][0]["operator"] == "quadratic"
    assert doc["factors"][0]["vars"] == [0]
    assert doc["factors"][0]["rho"] == [1.0]


def _doc():
    return json.loads(fg.serialize(two_quadratic_graph()))


@pytest.mark.parametrize("mutate,match", [
    (lambda d: "{not json", "malformed graph document"),
    (lambda d: dict(d, version="other-v9"), "version"),
    (lambda d: {"version": fg.DOCUMENT_VERSION, "factors": []}, "variables"),
    (lambda d: (d["variables"][0].update(id=7), d)[1], "contiguous"),
    (lambda d: (d["factors"][0].update(operator="warp_drive"), d)[1], "warp_drive"),
    (lambda d: (d["factors"][0].update(vars=[3]), d)[1], "unknown variable 3"),
])
def test_deserialize_rejections(mutate, match):
    """test_graph.py:162-196: the six malformed-document cases."""
    d = mutate(_doc())
    text = d if isinstance(d, str) else json.dumps(d)
    with pytest.raises(ValueError, match=match):
        fg.deserialize(text)


# ---------------------------------------------------------------------------
# reference FactorGraph objects through this package's plan builder

LAYOUT = ("edge_var", "edge_offsets", "var_offsets", "zmap", "z_weights", "rho_flat",
          "alpha_flat", "edge_rho", "edge_alpha", "edge_factor")


def _pairs(ref):
    P = ref.problems
    rng = np.random.default_rng(0)
    A = 0.05 * rng.standard_normal((16, 16))
    B = 0.1 * rng.standard_normal((16, 4))
    q0 = rng.standard_normal(16)
    pts = P.gen_gaussian_data(300, 32, 4.0, seed=0)
    X, y = fg.gen_gaussian_arrays(300, 32, 4.0, seed=0)
    return [
        ("pack", P.build_packing(P.PackingSpec(40)), fg.build_packing(fg.PackingSpec(40))),
        ("svm", P.build_svm(P.SvmSpec(pts, lam=1.0)),
         fg.build_svm(fg.SvmSpec.from_arrays(X, y, lam=1.0))),
        ("mpc", P.build_mpc(P.MpcSpec(60, ref.LinearSystem(A, B), q0)),
         fg.build_mpc(fg.MpcSpec(60, fg.LinearSystem(A, B), q0))),
    ]


def _same(a, b, what):
    if a is None or b is None:
        assert a is None and b is None, what
    else:
        np.testing.assert_array_equal(np.asarray(a), np.asarray(b), err_msg=what)


@pytest.mark.reference
def test_reference_factorgraph_same_groups_and_layout():
    ref = import_reference()
    import fgadmm.problems  # noqa: F401
    for name, rg, og in _pairs(ref):
        for key in LAYOUT:
            ra = np.asarray(getattr(rg, key))
            oa = np.asarray(getattr(og, key))
            np.testing.assert_array_equal(ra, oa, err_msg=f"{name}.{key}")
        assert rg.total_edge_payload == og.total_edge_payload
        assert rg.z_dim == og.z_dim
        rs, os_ = _group_specs(rg), _group_specs(og)
        assert [(c.kind, d) for c, d, *_ in rs] == [(c.kind, d) for c, d, *_ in os_], name
        for (rc, rd, rfe, rdp, _rp, _rsz), (oc, od, ofe, odp, _op, _osz) in zip(rs, os_):
            what = f"{name}/{rc.kind}"
            np.testing.assert_array_equal(rfe, ofe, err_msg=what + " first edges")
            _same(rdp.fparams, odp.fparams, what + " fparams")
            _same(rdp.tables, odp.tables, what + " tables")
            _same(rdp.fsys, odp.fsys, what + " fsys")
            assert rdp.iparam == odp.iparam, what


@pytest.mark.reference
@pytest.mark.parametrize("tag", DOCS)
def test_reference_deserialize_equals_ours(tag):
    ref = import_reference()
    doc = read_doc(tag)
    rg, og = ref.deserialize(doc), fg.deserialize(doc)
    for key in LAYOUT:
        np.testing.assert_array_equal(np.asarray(getattr(rg, key)),
                                      np.asarray(getattr(og, key)), err_msg=key)
