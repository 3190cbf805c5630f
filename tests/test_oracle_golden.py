"""Pin the CPU oracle (oracle/twostage_oracle.py) on the reference's own
outputs (tests/golden/golden.npz, made by tests/golden/make_golden.py from
the real `orthoqr` package) and on SPEC.md's known-answer examples.

The oracle is only trusted as the GPU parity checker once this passes.
"""
import numpy as np
import pytest

from oracle import twostage_oracle as O
from paper_2602_14449_b200 import workloads as W


def rel(x, y):
    x, y = np.asarray(x), np.asarray(y)
    d = np.abs(x - y).max() if x.size else 0.0
    return d / max(np.abs(y).max(), 1e-300) if y.size else 0.0


def cases(golden, prefix_filter=None):
    keys = sorted({k.rsplit("/", 1)[0] for k in golden.files if k.endswith("/q")})
    return [k for k in keys if prefix_filter is None or k.startswith(prefix_filter)]


def test_rand_stream_bitexact(golden):
    assert np.array_equal(W.normal_matrix(W.make_rng(12345), 7, 5), golden["rand/real/x"])
    assert np.array_equal(W.normal_matrix(W.make_rng(99), 4, 3, "complex"),
                          golden["rand/complex/x"])
    assert np.array_equal(W.uniform(W.make_rng(43), 0.0, 4.0, 9), golden["rand/uniform/x"])


TWO_STAGE_GROUPS = ["eq12", "eye", "real_", "cholshift", "cplx_", "rankdef"]


@pytest.mark.parametrize("group", TWO_STAGE_GROUPS)
def test_two_stage_matches_reference(golden, group):
    n_checked = 0
    for case in cases(golden, group):
        base = case.rsplit("/", 1)[0]
        v, a = golden[base + "/v"], golden[base + "/a"]
        choice = str(golden[case + "/choice"])
        intra = str(golden[case + "/intra"])
        p = golden[case + "/p"]
        out = O.two_stage(v, a, choice, intra, p if p.size else None)
        tol = 1e-11
        if group == "rankdef":
            # elementwise parity is meaningless on rank-deficient input
            # (SURVEY §8(c)); compare stability metrics instead
            loss, cross, res = O.stability(v, a, out["q"], out["r"], out["s"])
            assert loss <= 10 * max(float(golden[case + "/loss"]), 1e-15)
            assert res <= 10 * max(float(golden[case + "/resid"]), 1e-15)
        else:
            assert rel(out["q"], golden[case + "/q"]) < tol, case
            assert rel(out["r"], golden[case + "/r"]) < tol, case
            assert rel(out["s"], golden[case + "/s"]) < tol, case
        assert abs(out["kappa_t"] - float(golden[case + "/kappa_t"])) <= 1e-10 * float(golden[case + "/kappa_t"])
        assert abs(out["wt_inv_norm"] - float(golden[case + "/wt_inv_norm"])) <= 1e-10 * float(golden[case + "/wt_inv_norm"])
        n_checked += 1
    assert n_checked > 0


def test_eq12_two_u(golden):
    # PAPER.md:810-816 / SPEC.md acceptance 1: loss <= 1e-15 for all choices
    for ch in ("mlu", "qr", "polar"):
        assert float(golden[f"eq12/{ch}/loss"]) <= 1e-15
        v, a = golden["eq12/v"], golden["eq12/a"]
        out = O.two_stage(v, a, ch)
        loss, _, _ = O.stability(v, a, out["q"], out["r"], out["s"])
        assert loss <= 1e-15
        assert np.allclose(out["r"], np.diag([1e-30, 1e-30]), rtol=1e-12, atol=0)


def test_degenerate(golden):
    out = O.two_stage(np.zeros((50, 0)), golden["k0zero/a"])
    assert rel(out["q"], golden["k0zero/q"]) < 1e-13 and out["s"].shape == (0, 3)
    out = O.two_stage(golden["kzero/v"], np.zeros((50, 0)))
    assert out["q"].shape == (50, 0) and out["s"].shape == (4, 0)


def test_householder_qr(golden):
    for nn in (0, 1):
        q, r = O.lapack_qr(golden[f"hqr/nonneg{nn}/a"], nonneg=bool(nn))
        assert rel(q, golden[f"hqr/nonneg{nn}/q"]) < 1e-13
        assert rel(r, golden[f"hqr/nonneg{nn}/r"]) < 1e-13
    q, r = O.lapack_qr(np.array([[3.0], [4.0]]))
    assert np.allclose(q[:, 0], [-0.6, -0.8]) and np.isclose(r[0, 0], -5.0)
    q, r = O.lapack_qr(np.array([[3.0], [4.0]]), nonneg=True)
    assert np.allclose(q[:, 0], [0.6, 0.8]) and np.isclose(r[0, 0], 5.0)


def test_modified_lu(golden):
    for tag in ("zero", "diag", "rand"):
        p, lo, up = O.mlu(golden[f"mlu/{tag}/z"])
        assert np.array_equal(p, golden[f"mlu/{tag}/p"])
        assert rel(lo, golden[f"mlu/{tag}/l"]) < 1e-13
        assert rel(up, golden[f"mlu/{tag}/u"]) < 1e-13
    p, lo, up = O.mlu(np.zeros((3, 3)))
    assert np.array_equal(p, -np.ones(3)) and np.array_equal(up, -np.eye(3))
    with pytest.raises(O.OracleError) as ei:
        O.mlu(np.eye(3) * 1.5)
    assert ei.value.kind == "NormBoundError"


def test_reflector_pieces(golden):
    for ch in ("mlu", "qr", "polar"):
        h = O.Reflector(golden[f"refl/{ch}/v"], ch)
        assert rel(h.p, golden[f"refl/{ch}/p"]) < 1e-12
        assert rel(h.w[:10], golden[f"refl/{ch}/wtop"]) < 1e-12
        assert rel(h.tf.dense(), golden[f"refl/{ch}/t"]) < 1e-12
        kt, wn = h.diagnostics()
        assert abs(kt - float(golden[f"refl/{ch}/kappa_t"])) < 1e-11 * kt
        assert abs(wn - float(golden[f"refl/{ch}/wt_inv_norm"])) < 1e-11 * wn


def test_binner(golden):
    for tag in ("binner_dense", "binner_diag_real", "binner_diag_complex"):
        for ch in ("mlu", "qr", "polar"):
            g = lambda k: golden[f"{tag}/{ch}/{k}"]
            if tag == "binner_dense":
                ip = O.BInner(b=g("b"))
            else:
                ip = O.BInner(diag=g("d"))
            out = O.b_two_stage(g("v"), g("a"), g("u"), ip, ch)
            for key in ("q", "r", "s"):
                assert rel(out[key], g(key)) < 1e-9, (tag, ch, key)
            assert abs(out["kappa_t"] - float(g("kappa_t"))) < 1e-10 * float(g("kappa_t"))


def test_block_driver(golden):
    a = golden["block/a"]
    q, r = O.block_qr([a[:, i:i + 6] for i in range(0, 24, 6)])
    assert rel(q, golden["block/q"]) < 1e-11 and rel(r, golden["block/r"]) < 1e-11


def test_errors(golden):
    with pytest.raises(O.OracleError) as ei:
        O.two_stage(golden["err/orth/v"], np.ones((60, 2)))
    assert ei.value.kind == "OrthonormalityError"
    assert str(ei.value) == str(golden["err/orth/msg"])
    with pytest.raises(O.OracleError) as ei:
        O.two_stage(np.eye(5, 3), np.ones((5, 3)))
    assert ei.value.kind == "DimensionError"
