"""The oracle's operator READINGS pinned against an independent transcription
(tests/definitional.py, numpy binary32 + exactly rounded fma, written from SURVEY.md
§8(c) / DESIGN.md §3), bit for bit on ~10^4 inputs per function.

Accuracy bounds (test_oracle_math / test_oracle_rowops) admit neighbouring op orders;
these tests do not: each one also shows that a plausible alternative reading (divide
instead of reciprocal-multiply, unfused LN affine, a coefficient off by one ulp, a
sequential instead of a 128-slot sum) differs from the oracle on the same inputs, so
the comparison has the power to catch that drift."""
import numpy as np
import pytest

from tests import definitional as D
from tests import ieee_sim
import oracle
import synth


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def assert_same(got, ref, what):
    g, r = bits(got).ravel(), bits(ref).ravel()
    bad = np.flatnonzero(g != r)
    assert bad.size == 0, f"{what}: {bad.size}/{g.size} differ, first {bad[:4]} oracle {g[bad[:4]]} def {r[bad[:4]]}"


def ulp_step(x, k=1):
    return (np.array([x], np.float32).view(np.uint32) + np.uint32(k)).view(np.float32)[0]


# ---------------------------------------------------------------------- the exact fma itself
def test_fma32_matches_exact_rational_model():
    rng = np.random.default_rng(0)
    n = 4000
    a = synth.uniform(1, n, 4.0)
    b = synth.uniform(2, n, 4.0)
    c = synth.uniform(3, n, 16.0)
    # ties and near-ties: a = b = 1 + 2^-12 (product needs 25 bits), c = -1 etc.; subnormal range; cancellation
    a[:8] = b[:8] = np.float32(1 + 2.0 ** -12)
    c[:8] = np.float32([-1, 1, -2 ** -24, 2 ** -24, 0, -0.0, 3, -3])
    a[8:40] = (a[8:40] * np.float32(2.0 ** -70)).astype(np.float32)
    b[8:40] = (b[8:40] * np.float32(2.0 ** -70)).astype(np.float32)
    c[8:40] = (c[8:40] * np.float32(2.0 ** -140)).astype(np.float32)
    c[40:80] = -(a[40:80].astype(np.float64) * b[40:80]).astype(np.float32)   # near-total cancellation
    a[80:90] = np.float32(2.0 ** 100)
    b[80:90] = np.float32(2.0 ** 28)                                            # overflow to inf
    idx = rng.permutation(n)[:1500].tolist() + list(range(90))
    got = D.fma32(a[idx], b[idx], c[idx])
    ref = np.array([ieee_sim.fma(a[i], b[i], c[i]) for i in idx], np.float32)
    assert_same(got, ref, "fma32 vs exact rational")
    # and it is not the double-rounded a*b+c in float64
    assert np.float32(np.float64(a[0]) * b[0] + np.float64(c[0])) == D.fma32(a[0], b[0], c[0])  # (a tie-free case)
    assert D.fma32(np.float32(1 + 2.0 ** -12), np.float32(1 + 2.0 ** -12), np.float32(-1)) == \
        np.float32(2.0 ** -11 + 2.0 ** -24)


# ---------------------------------------------------------------------- elementwise math
def _inputs(tag, lo, hi, n=12000):
    x = (synth.uniform(synth.seed_for("def", tag), n, 1.0) * np.float32((hi - lo) / 2) +
         np.float32((hi + lo) / 2)).astype(np.float32)
    return x


def test_exp_reading():
    x = np.concatenate([_inputs("exp", -104, 89), _inputs("exp2", -2, 2),
                        np.float32([0, -0.0, 1, -1, 88.72283172607422, 88.72283935546875, 89, 89.5, -103.9, -104,
                                    -104.5, np.inf, -np.inf, np.nan, 1e-30, -87.5, -95, -100, -87.33654]),
                        (_inputs("exp3", -1, 1) * np.float32(1e-6)).astype(np.float32)])
    ref = D.exp(x)
    assert_same(oracle.exp(x), ref, "R-EXP")
    assert bits(D.exp(np.float32([1.0])))[0] == 0x402DF854  # exp(1) correctly rounded (paper-independent pin)


def test_log_reading_and_coefficient_power():
    x = np.concatenate([np.abs(_inputs("log", -1000, 1000)), np.abs(_inputs("log2", -2, 2)),
                        np.float32([1, 2, 0.5, 0.7071067, 0.70710677, 0.7071068, 3.4e38, 1e-38, 1e-40, 1.4e-45, 0,
                                    -0.0, -1, np.inf, np.nan])])
    ref = D.log(x)
    assert_same(oracle.log(x), ref, "R-LOG")
    # power: perturbing any polynomial coefficient (as a binary32 constant) is caught by
    # these inputs -- the low-order ones at 1 ulp; the high-order ones multiply f^6..f^9
    # (|f| < 0.3), so only a change of 4-256 ulps of the constant reaches an output bit
    # (a smaller change is bit-invisible, i.e. it defines the same function on these inputs)
    thresholds = (256, 32, 32, 4, 1, 1, 1, 1)
    for i, k in enumerate(thresholds):
        co = list(D.LOG_C)
        co[i] = float(ulp_step(np.float32(co[i]), k))
        assert np.any(bits(D.log(x, co)) != bits(ref)), f"coefficient {i} (+{k} ulp) not discriminated"


@pytest.mark.parametrize("fn", ["exp", "log", "tanh", "gelu"])
def test_strided_sweep_of_all_binary32(fn):
    # every 257th bit pattern of all 2^32 (16.7 M inputs: every exponent, both signs,
    # subnormals, infinities and NaNs)
    u = np.arange(0, 2 ** 32, 257, dtype=np.uint64).astype(np.uint32)
    x = u.view(np.float32)
    assert_same(getattr(oracle, fn)(x), getattr(D, fn)(x), f"{fn} strided sweep")


def test_tanh_reading():
    x = np.concatenate([_inputs("tanh", -12, 12), _inputs("tanh2", -0.7, 0.7),
                        np.float32([0, -0.0, 0.625, 0.62499994, -0.625, 44, 50, -50, 1e-20, np.inf, -np.inf,
                                    np.nan])])
    assert_same(oracle.tanh(x), D.tanh(x), "R-TANH")


def test_gelu_forward_backward_reading():
    x = np.concatenate([_inputs("gelu", -8, 8), _inputs("gelu2", -0.5, 0.5), np.float32([0, -0.0, 3, -3, 10])])
    dy = synth.uniform(7, x.size, 2.0)
    assert_same(oracle.gelu(x), D.gelu(x), "R-GELU")
    assert_same(oracle.gelu_backward(x, dy), D.gelu_backward(x, dy), "R-GELU bwd")


# ---------------------------------------------------------------------- reductions
def test_csum_cdot_reading_and_alternatives():
    for n in (1, 127, 128, 129, 1000, 4096, 4097, 9000, 50257):
        x = synth.uniform(synth.seed_for("dcs", n), n, 3.0)
        x[: min(n, 3)] *= np.float32(2.0 ** 20)
        y = synth.uniform(synth.seed_for("dcd", n), n, 3.0)
        assert bits(oracle.csum(x)) == bits(D.csum(x)), n
        assert bits(oracle.cdot(x, y)) == bits(D.cdot(x, y)), n
    x = synth.uniform(synth.seed_for("dcs", 50257), 50257, 3.0)
    seqsum = np.float32(0)
    for v in x:
        seqsum = np.float32(seqsum + v)
    assert bits(seqsum) != bits(D.csum(x))  # the sequential reading differs on this input


# ---------------------------------------------------------------------- row operators
def test_softmax_forward_backward_reading():
    rows, cols = 48, 320
    x = synth.uniform(11, (rows, cols), 6.0)
    ref = np.stack([D.softmax_row(x[r]) for r in range(rows)])
    assert_same(oracle.softmax(x), ref, "R-SOFTMAX")
    # causal rows (row r keeps (r mod cols) + 1 entries)
    xc = synth.uniform(12, (2 * 64, 64), 6.0)
    refc = np.stack([D.softmax_row(xc[r], valid=(r % 64) + 1) for r in range(xc.shape[0])])
    assert_same(oracle.softmax(xc, causal=True), refc, "R-SOFTMAX causal")
    # power: y = e / s (per-element divide) differs from the reciprocal-multiply reading
    alt = []
    for r in range(rows):
        e = D.exp(D.fsub(x[r], np.max(x[r])))
        alt.append(D.fdiv(e, D.csum(e)))
    assert np.any(bits(np.stack(alt)) != bits(ref))
    dy = synth.uniform(13, (rows, cols), 1.0)
    refb = np.stack([D.softmax_backward_row(ref[r], dy[r], 0.125) for r in range(rows)])
    assert_same(oracle.softmax_backward(ref, dy, scale=0.125), refb, "R-SOFTMAX bwd")


def test_layernorm_forward_backward_reading():
    rows, cols = 40, 768
    x = synth.uniform(21, (rows, cols), 3.0)
    x[:, :5] += np.float32(5.0)
    g = synth.uniform(22, cols, 2.0)
    b = synth.uniform(23, cols, 1.0)
    outs = [D.layernorm_row(x[r], g, b) for r in range(rows)]
    y, mu, rs = oracle.layernorm(x, g, b)
    assert_same(y, np.stack([o[0] for o in outs]), "R-LN y")
    assert_same(mu, np.array([o[1] for o in outs], np.float32), "R-LN mean")
    assert_same(rs, np.array([o[2] for o in outs], np.float32), "R-LN rstd")
    # power: the unfused affine fadd(fmul(xh, g), b) differs
    alt = []
    for r in range(rows):
        xh = D.fmul(D.fsub(x[r], outs[r][1]), outs[r][2])
        alt.append(D.fadd(D.fmul(xh, g), b))
    assert np.any(bits(np.stack(alt)) != bits(y))
    dy = synth.uniform(24, (rows, cols), 1.0)
    dres = synth.uniform(25, (rows, cols), 1.0)
    refdx = np.stack([D.layernorm_backward_row(dy[r], x[r], g, mu[r], rs[r], dres[r]) for r in range(rows)])
    assert_same(oracle.layernorm_backward(dy, x, g, mu, rs, dres=dres), refdx, "R-LN bwd")
    refdx0 = np.stack([D.layernorm_backward_row(dy[r], x[r], g, mu[r], rs[r]) for r in range(rows)])
    assert_same(oracle.layernorm_backward(dy, x, g, mu, rs), refdx0, "R-LN bwd (no residual)")
    dg, db = oracle.layernorm_backward_params(dy, x, mu, rs)
    rg, rb = D.layernorm_params(dy, x, mu, rs)
    assert_same(dg[0], rg, "R-LN dgamma")
    assert_same(db[0], rb, "R-LN dbeta")


def test_cross_entropy_reading():
    rows, V = 12, 5003
    x = synth.uniform(31, (rows, V), 8.0)
    lab = synth.integers(32, rows, V).astype(np.int32)
    loss, dl = oracle.cross_entropy(x, lab, scale=2.0 ** -12)
    for r in range(rows):
        l_r, d_r = D.cross_entropy_row(x[r], int(lab[r]), 2.0 ** -12)
        assert bits(loss[r]) == bits(l_r), r
        assert_same(dl[r], d_r, f"R-CE grad row {r}")


def test_adamw_reading():
    n = 10000
    p = synth.uniform(41, n, 0.05)
    g = synth.uniform(42, n, 1e-3)
    g[:10] = np.float32([0, -0.0, 1e-30, -1e-30, 1, -1, 1e-8, 3e-4, -7e-5, 2.0 ** -126])
    m = synth.uniform(43, n, 1e-4)
    v = np.abs(synth.uniform(44, n, 1e-6))
    for step, decay in ((1, True), (1, False), (7, True)):
        ref = D.adamw(p, g, m, v, step, 6e-4, 0.9, 0.95, 1e-8, 0.1, decay)
        got = oracle.adamw(p, g, m, v, step, 6e-4, 0.9, 0.95, 1e-8, 0.1, decay)
        for a, b_, w in zip(got, ref, ("p'", "m'", "v'")):
            assert_same(a, b_, f"R-ADAMW {w} step {step} decay {decay}")
