"""Next-token sampling (vqb_sample, the C5 decode loop's last step) against the CPU
restatement in oracle/sample_oracle.py: greedy = torch.argmax (lowest index on
ties), temperature / top-k Gumbel-max draws = the oracle's token up to fp32 score
rounding (1e-4 on the oracle's float64 scores), the top-k set (ties at the k-th
value kept), the top-p nucleus (fp32 fixed-point weights: 2e-3 mass margin), and the
sampled distribution = softmax(logits / T) over the kept set."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import sample_oracle as SO  # noqa: E402


def test_oracle_uniform_range_and_moments():
    u = SO.uniform(7, 3, 1, np.arange(200000))
    assert u.min() > 0 and u.max() < 1
    assert abs(u.mean() - 0.5) < 0.005 and abs(u.var() - 1 / 12) < 0.002
    assert not np.array_equal(u[:100], SO.uniform(7, 4, 1, np.arange(100)))  # the step changes the draw


def test_oracle_top_k_keeps_ties():
    lg = np.array([[1.0, 3.0, 2.0, 2.0, 0.5]])
    assert SO.keep_mask(lg, 2).tolist() == [[False, True, True, True, False]]
    assert SO.keep_mask(lg, 0).all() and SO.keep_mask(lg, 5).all()


@pytest.fixture(scope="module")
def dev():
    return torch.device("cuda", 0)


def _chosen_ok(tok, sc):
    best = sc.max(axis=1)
    got = sc[np.arange(len(tok)), tok]
    return np.all(np.isfinite(got)) and np.all(got >= best - 1e-4 * np.maximum(1.0, np.abs(best)))


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float16, torch.float32])
def test_greedy_matches_argmax(dtype, dev):
    from paper_2503_02236_b200 import _native as N
    from paper_2503_02236_b200 import ops
    g = torch.Generator(device=dev).manual_seed(1)
    lg = (torch.randn((9, 32000), generator=g, device=dev) * 3).to(dtype)
    lg[3, 100] = lg[3, 31000] = lg[3].max() + 1  # tie: the lowest index wins
    tok = ops.sample(lg)
    assert N.last_kernel() == "sample"
    assert torch.equal(tok, torch.argmax(lg, dim=-1))
    assert int(tok[3]) == 100


@pytest.mark.gpu
@pytest.mark.parametrize("temperature,top_k", [(1.0, 0), (0.7, 0), (1.3, 50), (1.0, 1), (2.0, 31999)])
def test_draw_matches_oracle(temperature, top_k, dev):
    from paper_2503_02236_b200 import ops
    g = torch.Generator(device=dev).manual_seed(2)
    lg = (torch.randn((32, 32000), generator=g, device=dev) * 2).half()
    step = torch.tensor([57], dtype=torch.int32, device=dev)
    tok = ops.sample(lg, temperature, top_k, seed=123, d_step=step).cpu().numpy()
    host = lg.float().cpu().numpy()
    sc = SO.scores(host, temperature, top_k, 123, 57)
    assert _chosen_ok(tok, sc)
    want = SO.sample(host, temperature, top_k, 123, 57)
    assert (tok == want).mean() >= 0.95  # exact but for fp32 near-ties
    if top_k == 1:
        assert np.array_equal(tok, host.argmax(axis=1))


@pytest.mark.gpu
def test_top_k_set_with_ties(dev):
    from paper_2503_02236_b200 import ops
    v = 4096
    base = torch.full((v,), -5.0)
    base[[10, 20, 30, 40]] = torch.tensor([4.0, 3.0, 2.0, 2.0])  # k = 3: the tie at 2.0 keeps both
    lg = base.repeat(2048, 1).to(dev)
    tok = ops.sample(lg, 5.0, 3, seed=9).cpu().numpy()
    assert set(np.unique(tok)) <= {10, 20, 30, 40}
    assert {30, 40} <= set(np.unique(tok))


@pytest.mark.gpu
def test_distribution_matches_softmax(dev):
    """20000 rows of the same 8 logits (each row hashes differently): frequencies
    within 5 sigma of softmax(l / T), and of the renormalised top-3 softmax."""
    from paper_2503_02236_b200 import ops
    l8 = torch.tensor([0.1, 1.5, -0.7, 0.9, 2.2, -2.0, 0.0, 1.1])
    rows = 20000
    lg = l8.repeat(rows, 1).to(dev)
    for temperature, k in ((1.0, 0), (0.5, 0), (1.5, 3)):
        tok = ops.sample(lg, temperature, k, seed=31).cpu().numpy()
        p = torch.softmax(l8 / temperature, 0).numpy().astype(np.float64)
        if k:
            keep = SO.keep_mask(l8.numpy()[None], k)[0]
            p = np.where(keep, p, 0.0)
            p /= p.sum()
        freq = np.bincount(tok, minlength=8) / rows
        sigma = np.sqrt(p * (1 - p) / rows) + 1e-12
        assert np.all(np.abs(freq - p) <= 5 * sigma + 1e-9), (temperature, k, freq, p)


@pytest.mark.gpu
def test_step_and_seed_determinism(dev):
    from paper_2503_02236_b200 import ops
    g = torch.Generator(device=dev).manual_seed(4)
    lg = torch.randn((16, 32000), generator=g, device=dev).half()
    s0 = torch.tensor([5], dtype=torch.int32, device=dev)
    s1 = torch.tensor([6], dtype=torch.int32, device=dev)
    a = ops.sample(lg, 1.0, 0, seed=1, d_step=s0)
    assert torch.equal(a, ops.sample(lg, 1.0, 0, seed=1, d_step=s0))
    assert not torch.equal(a, ops.sample(lg, 1.0, 0, seed=1, d_step=s1))
    assert not torch.equal(a, ops.sample(lg, 1.0, 0, seed=2, d_step=s0))


@pytest.mark.gpu
def test_sample_errors(dev):
    from paper_2503_02236_b200 import ops
    from paper_2503_02236_b200.errors import ConfigError, ShapeError
    lg = torch.zeros((2, 10), device=dev)
    with pytest.raises(ConfigError):
        ops.sample(lg, -1.0)
    with pytest.raises(ShapeError):
        ops.sample(lg.to(torch.int32))


def test_oracle_nucleus_mask():
    lg = np.array([[3.0, 2.0, 1.0, 0.0], [2.0, 2.0, 1.0, -5.0]])
    keep = np.ones(lg.shape, bool)
    assert SO.nucleus_mask(lg, 1.0, keep, 0.8)[0].tolist() == [True, True, False, False]
    assert SO.nucleus_mask(lg, 1.0, keep, 0.5)[0].tolist() == [True, False, False, False]
    assert SO.nucleus_mask(lg, 1.0, keep, 0.3)[1].tolist() == [True, True, False, False]  # ties kept
    assert SO.nucleus_mask(lg, 1.0, keep, 1.0).all()


@pytest.mark.gpu
@pytest.mark.parametrize("temperature,top_k,top_p", [(1.0, 0, 0.9), (0.7, 50, 0.8), (1.3, 0, 0.5)])
def test_nucleus_draw_matches_oracle(temperature, top_k, top_p, dev):
    from paper_2503_02236_b200 import ops
    g = torch.Generator(device=dev).manual_seed(12)
    lg = (torch.randn((32, 32000), generator=g, device=dev) * 3).half()
    step = torch.tensor([9], dtype=torch.int32, device=dev)
    tok = ops.sample(lg, temperature, top_k, seed=5, d_step=step, top_p=top_p).cpu().numpy()
    host = lg.float().cpu().numpy()
    t32 = float(np.float32(temperature))
    wide = SO.nucleus_mask(host, t32, SO.keep_mask(host, top_k), min(1.0, top_p + 2e-3))
    assert wide[np.arange(32), tok].all()  # every draw inside the nucleus (fp32 weights: small margin)
    want = SO.sample(host, temperature, top_k, 5, 9, top_p)
    assert (tok == want).mean() >= 0.9


@pytest.mark.gpu
def test_nucleus_distribution(dev):
    """Frequencies within 5 sigma of softmax renormalised over the nucleus."""
    from paper_2503_02236_b200 import ops
    l8 = torch.tensor([0.1, 1.5, -0.7, 0.9, 2.2, -2.0, 0.0, 1.1])
    rows = 20000
    lg = l8.repeat(rows, 1).to(dev)
    for temperature, top_p in ((1.0, 0.7), (0.6, 0.9)):
        tok = ops.sample(lg, temperature, 0, seed=17, top_p=top_p).cpu().numpy()
        keep = SO.nucleus_mask(l8.numpy()[None].astype(np.float64), temperature, np.ones((1, 8), bool), top_p)[0]
        p = torch.softmax(l8 / temperature, 0).numpy().astype(np.float64)
        p = np.where(keep, p, 0.0)
        p /= p.sum()
        freq = np.bincount(tok, minlength=8) / rows
        sigma = np.sqrt(p * (1 - p) / rows) + 1e-12
        assert np.all(np.abs(freq - p) <= 5 * sigma + 1e-9), (temperature, top_p, freq, p)


@pytest.mark.gpu
def test_top_p_errors(dev):
    from paper_2503_02236_b200 import ops
    from paper_2503_02236_b200.errors import ConfigError
    lg = torch.zeros((2, 10), device=dev)
    for bad in (0.0, 1.5):
        with pytest.raises(ConfigError):
            ops.sample(lg, 1.0, top_p=bad)
