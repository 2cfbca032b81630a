"""CPU ORACLE — TEST INFRASTRUCTURE ONLY (same import rule as vq_oracle.py).

Restates the decode loop's next-token draw (csrc/decode.cu sample_kernel,
include/vqb.h vqb_sample) so tests can check the kernel. vqforge has no sampler
(it stops at single fused kernels, SURVEY.md §8f row 1 adds one), so there is no
reference to pin against: the contract is the published Gumbel-max identity
(argmax_i(l_i / T + G_i), G_i standard Gumbel, is a draw from softmax(l / T)) and
the usual top-k warper rule (keep logits >= the k-th largest, ties kept).
Scores are computed in float64; the kernel uses fp32 and fast logarithms, so
tests compare chosen tokens through their oracle scores, not bit for bit.
"""

import numpy as np

_M64 = (1 << 64) - 1


def uniform(seed: int, step: int, row: int, idx: np.ndarray) -> np.ndarray:
    """u in (0, 1) of the counter hash (splitmix64 finaliser of seed, step, row, i)."""
    with np.errstate(over="ignore"):
        key = np.uint64(((int(seed) & _M64) ^ ((((int(step) & 0xFFFFFFFF) << 32) | (int(row) & 0xFFFFFFFF))
                                              * 0x9E3779B97F4A7C15 & _M64)))
        z = key + (idx.astype(np.uint64) + np.uint64(1)) * np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(30)
        z *= np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return ((z >> np.uint64(41)).astype(np.float64) + 0.5) / float(1 << 23)


def keep_mask(logits: np.ndarray, top_k: int) -> np.ndarray:
    """Logits >= the top_k-th largest (all when top_k is 0 or >= vocab)."""
    if top_k <= 0 or top_k >= logits.shape[-1]:
        return np.ones(logits.shape, bool)
    kth = -np.sort(-logits, axis=-1)[..., top_k - 1:top_k]
    return logits >= kth


def nucleus_mask(logits: np.ndarray, temperature: float, keep: np.ndarray, top_p: float) -> np.ndarray:
    """Within `keep`, the logits >= the largest threshold whose probability mass
    (softmax(logits / T) over `keep`) is >= top_p (ties at the threshold kept)."""
    if top_p >= 1.0:
        return keep
    out = np.zeros_like(keep)
    for b in range(logits.shape[0]):
        x = np.where(keep[b], logits[b].astype(np.float64), -np.inf)
        w = np.exp((x - x.max()) / temperature)
        order = np.argsort(-x, kind="stable")
        cum = np.cumsum(w[order])
        k = int(np.searchsorted(cum, top_p * cum[-1]))  # first prefix reaching the mass
        tau = x[order[min(k, len(order) - 1)]]
        out[b] = keep[b] & (x >= tau)
    return out


def scores(logits: np.ndarray, temperature: float, top_k: int, seed: int, step: int,
           top_p: float = 1.0) -> np.ndarray:
    """(B, V) float64 Gumbel-max scores, -inf outside the top-k / top-p set;
    temperature 0 = the logits themselves (greedy)."""
    lg = np.asarray(logits, np.float64)
    if temperature <= 0:
        return lg.copy()
    idx = np.arange(lg.shape[1])
    g = np.stack([-np.log(-np.log(uniform(seed, step, b, idx))) for b in range(lg.shape[0])])
    s = lg / np.float64(np.float32(temperature)) + g
    keep = nucleus_mask(lg, float(np.float32(temperature)), keep_mask(lg, top_k), top_p)
    return np.where(keep, s, -np.inf)


def sample(logits: np.ndarray, temperature: float, top_k: int, seed: int, step: int,
           top_p: float = 1.0) -> np.ndarray:
    """Next tokens (B,) int64: argmax of scores, lowest index on ties."""
    return np.argmax(scores(logits, temperature, top_k, seed, step, top_p), axis=1).astype(np.int64)
