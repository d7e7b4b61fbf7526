"""Pins of the config-1 oracle pieces: ReLU (reading R24) and the
whole MLP step (oracle/mlp_step.py) against float64 mathematics: forward values,
gradients by central finite differences of the float64 loss, the shard combine,
and loss decrease after the AdamW update."""
from dataclasses import dataclass

import numpy as np
import pytest

import oracle
import synth
from oracle import mlp_step


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def test_relu_spec_examples_and_special_values():
    assert oracle.relu(np.float32([-1, 2])).tolist() == [0, 2]
    assert oracle.relu_backward(np.float32([-1, 2]), np.float32([5, 7])).tolist() == [0, 7]
    x = np.float32([-0.0, 0.0, np.inf, -np.inf, 1e-45, -1e-45, np.nan, 3.5])
    y = oracle.relu(x)
    assert bits(y).tolist() == bits(np.float32([0, 0, np.inf, 0, 1e-45, 0, np.nan, 3.5])).tolist()
    assert bits(y)[6] == 0x7FC00000                                                    # R10 canonical NaN
    g = np.float32([9, 9, 9, 9, 9, 9, 9, -2])
    d = oracle.relu_backward(x, g)
    assert bits(d).tolist() == bits(np.float32([0, 0, 9, 0, 9, 0, np.nan, -2])).tolist()  # subgradient 0 at 0


def test_relu_matches_numpy_where_and_finite_differences():
    x = synth.uniform(5, (8, 8))
    assert np.array_equal(bits(oracle.relu(x)), bits(np.where(x > 0, x, np.float32(0))))
    e = 1e-3
    x64 = x.astype(np.float64)
    x64 = np.where(np.abs(x64) < 2 * e, 0.5, x64)  # keep away from the kink
    fd = (np.maximum(x64 + e, 0) - np.maximum(x64 - e, 0)) / (2 * e)
    g = synth.uniform(6, (8, 8))
    got = oracle.relu_backward(x64.astype(np.float32), g)
    assert np.allclose(got, fd * g, rtol=1e-3, atol=1e-6)


@dataclass
class Cfg:
    batch: int = 32
    width: int = 256
    classes: int = 256
    shards: int = 8
    lr: float = 1e-2
    beta1: float = 0.9
    beta2: float = 0.95
    adam_eps: float = 1e-8
    wd: float = 0.1
    seed: int = 0


def loss64(p, x, y):
    h = x @ p["W1"] + p["b1"]
    a = np.maximum(h, 0)
    z = a @ p["W2"] + p["b2"]
    m = z.max(1, keepdims=True)
    lse = m[:, 0] + np.log(np.exp(z - m).sum(1))
    return (lse - z[np.arange(len(y)), y]).sum() / len(y)


@pytest.fixture(scope="module")
def step():
    cfg = Cfg()
    out, inp = mlp_step.run_step(cfg)
    return cfg, out, inp


def test_mlp_forward_close_to_float64(step):
    cfg, out, inp = step
    R = cfg.batch // cfg.shards
    for s in (0, 7):
        xs = inp["x"][s * R:(s + 1) * R].astype(np.float64)
        h = xs @ inp["W1"].astype(np.float64) + inp["b1"]
        assert np.allclose(out[f"s{s}/h"], h, rtol=1e-5, atol=1e-5)
        a = np.maximum(h, 0)
        z = a @ inp["W2"].astype(np.float64) + inp["b2"]
        assert np.allclose(out[f"s{s}/z"], z, rtol=1e-5, atol=1e-5)


def test_mlp_gradients_match_finite_differences(step):
    cfg, out, inp = step
    p64 = {n: inp[n].astype(np.float64) for n in mlp_step.PARAMS}
    x, y = inp["x"].astype(np.float64), inp["labels"]
    rng = np.random.default_rng(0)
    eps = 1e-4
    for n in mlp_step.PARAMS:
        g = out[f"grad/{n}"]
        for _ in range(6):
            idx = tuple(int(rng.integers(0, s)) for s in p64[n].shape)
            pp = {k: v.copy() for k, v in p64.items()}
            pm = {k: v.copy() for k, v in p64.items()}
            pp[n][idx] += eps
            pm[n][idx] -= eps
            fd = (loss64(pp, x, y) - loss64(pm, x, y)) / (2 * eps)
            assert abs(g[idx] - fd) <= 1e-3 * abs(fd) + 1e-6, (n, idx, g[idx], fd)


def test_mlp_shard_combine_and_update(step):
    cfg, out, inp = step
    for n in mlp_step.PARAMS:
        parts = np.stack([out[f"s{s}/grad/{n}"].astype(np.float64) for s in range(cfg.shards)])
        assert np.allclose(out[f"grad/{n}"], parts.sum(0), rtol=1e-6, atol=1e-9)
    x, y = inp["x"].astype(np.float64), inp["labels"]
    before = loss64({n: inp[n].astype(np.float64) for n in mlp_step.PARAMS}, x, y)
    after = loss64({n: out[f"param'/{n}"].astype(np.float64) for n in mlp_step.PARAMS}, x, y)
    assert after < before
    mean_loss = np.concatenate([out[f"s{s}/loss"] for s in range(cfg.shards)]).mean()
    assert abs(mean_loss - before) < 1e-5 * before
