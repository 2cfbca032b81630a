"""Hierarchical fusion: how dequantized codebook entries reach the consumer's
operand layout (paper §VI-B, Alg. 1; reference pkg/src/vqforge/fusion.py).

The reference decides between *register* fusion (intra-warp xor exchanges inside
mini-warps of ``v / required_layout`` lanes; ``n_shuffle = iters - 1``) and
*shared* fusion (stage the dequantized tile in shared memory) by comparing the
exchange count with the profiled latency ratio THRES_SHUFFLE. The schedule API
below reproduces its mapping and is verified lane by lane against the
reference's ownership oracle (tests/test_host.py).

On B200 the level selects a kernel family (``b200_fusion``):

* ``register`` — looked-up entries go straight into the consumer's registers:
  CUDA-core FMAs where a lane owns whole sub-vectors (GEMV batch 1-2, decode
  attention: zero exchanges needed), or mma.sync A fragments gathered by
  ``ldmatrix.trans`` from the replicated table (GEMV batch 4: the hardware
  transpose replaces the xor exchange schedule);
* ``shared`` — the dequantized W tile is written to shared memory in the UMMA
  canonical layout for tcgen05 (decode GEMV at 5-64 rows with the batch as the
  UMMA N, prefill GEMM): tcgen05.mma reads operands only from shared memory / TMEM.
"""

import json
from dataclasses import dataclass

import numpy as np

from .errors import MappingError

WARP = 32
THRES_SHUFFLE = 5
STYLE_STRIDED = "strided"
STYLE_MMA = "mma"
B200_GEMV_MAX_ROWS = 4  # rows above this take tcgen05 (shared-level fusion): the decode GEMV to 64 rows, then the GEMM
B200_GEMV_TC_MAX_ROWS = 64


def _pow2(n: int) -> bool:
    return n > 0 and (n & (n - 1)) == 0


@dataclass(frozen=True)
class LayoutPair:
    """Elements per thread after dequantization (src = v) and as the consumer needs them (dst)."""

    layout_src: int
    layout_dst: int

    def __post_init__(self):
        if not (_pow2(self.layout_src) and _pow2(self.layout_dst)):
            raise MappingError(f"layouts must be powers of two, got {self.layout_src}/{self.layout_dst}")

    @property
    def register_compatible(self) -> bool:
        return self.layout_dst <= self.layout_src

    @property
    def iters(self) -> int:
        if not self.register_compatible:
            raise MappingError(f"register fusion needs layout_src >= layout_dst "
                               f"({self.layout_src} < {self.layout_dst})")
        return self.layout_src // self.layout_dst

    @property
    def n_shuffle(self) -> int:
        return self.iters - 1


def shuffle_count(vector_size: int, required_layout: int) -> int:
    return LayoutPair(vector_size, required_layout).n_shuffle


def choose_fusion_level(layouts: LayoutPair, thres_shuffle: int = THRES_SHUFFLE) -> str:
    ok = layouts.register_compatible and layouts.n_shuffle < thres_shuffle
    return "register" if ok else "shared"


def b200_fusion(op_kind: str, rows: int = 1) -> str:
    """Fusion level of the sm_100a kernel that serves the op (see module doc): up to
    4 rows the lookups feed registers (CUDA cores / mma.sync); above, the dequantized
    W tile is staged in shared memory for tcgen05 (the decode GEMV with the batch as
    the UMMA N to 64 rows, the GEMM beyond)."""
    if rows > B200_GEMV_MAX_ROWS:
        return "shared"
    return "register"


@dataclass(frozen=True)
class WarpTile:
    rows: int
    cols: int
    style: str

    @property
    def n_elements(self) -> int:
        return self.rows * self.cols


def default_warp_tile(layouts: LayoutPair, style: str) -> WarpTile:
    """Strided: 32 rows of v. MMA (dst 2): 16 rows of 2v (one m16n8k16 A operand
    row pair per lane quad); below v = 4 the strided tile is used."""
    if style not in (STYLE_STRIDED, STYLE_MMA):
        raise MappingError(f"unknown compute style {style!r}")
    src = layouts.layout_src
    if style == STYLE_MMA:
        if layouts.layout_dst != 2:
            raise MappingError("mma consumers take layout_dst = 2")
        if src >= 4:
            return WarpTile(16, 2 * src, STYLE_MMA)
    return WarpTile(WARP, src, STYLE_STRIDED)


def compute_owner(tile: WarpTile, dst: int, e: np.ndarray):
    """(lane, slot) that consumes element e in the compute layout."""
    e = np.asarray(e)
    if tile.style == STYLE_STRIDED:
        return (e // dst) % WARP, e // (WARP * dst)
    r, c = np.divmod(e, tile.cols)
    return 4 * (r % 8) + (c % 8) // 2, (tile.cols // 8) * (r // 8) + c // 8


@dataclass(frozen=True)
class ShuffleSchedule:
    layouts: LayoutPair
    tile: WarpTile
    mini_warp_size: int
    thread_remap: tuple
    offsets: tuple

    @property
    def n_shuffle(self) -> int:
        return len(self.offsets)

    @property
    def subvector_of_lane(self) -> np.ndarray:
        """Inverse remap: the naive sub-vector each lane dequantizes."""
        return np.argsort(np.asarray(self.thread_remap))

    def to_json(self) -> str:
        return json.dumps({"mini_warp_size": self.mini_warp_size, "remap": list(self.thread_remap),
                           "offsets": list(self.offsets)})


def build_thread_mapping(warp_tile: WarpTile, layouts: LayoutPair) -> np.ndarray:
    """remap[sub-vector] = lane that dequantizes it, chosen so every xor-aligned
    mini-warp of ``iters`` lanes dequantizes exactly the elements it consumes."""
    src, it = layouts.layout_src, layouts.iters
    if it > WARP:
        raise MappingError(f"an exchange group of {it} lanes exceeds the warp; use shared fusion")
    consumer, _ = compute_owner(warp_tile, layouts.layout_dst, np.arange(warp_tile.n_elements))
    # consumer lanes of each sub-vector's src elements, as a (32, src) matrix
    cons = consumer.reshape(WARP, src)
    first = cons.min(axis=1)
    sig = np.sort(cons, axis=1)
    # each sub-vector must feed one complete xor-aligned group {g, g+1, ..., g+it-1},
    # met in ascending lane order along its elements
    for row in cons:
        _, at = np.unique(row, return_index=True)
        if np.any(np.diff(row[np.sort(at)]) < 0):
            raise MappingError("consumer lanes of a sub-vector are not met in ascending order; use shared fusion")
    groups = np.unique(sig, axis=0)
    for row in groups:
        lanes = np.unique(row)
        if lanes.size != it or lanes[0] % it or not np.array_equal(lanes, lanes[0] + np.arange(it)):
            raise MappingError(f"consumer lanes {lanes.tolist()} are not an aligned {it}-lane exchange "
                               "group; use shared fusion")
    # sub-vectors feeding a group are assigned to that group's lanes in order
    order = np.lexsort((np.arange(WARP), first))
    remap = np.empty(WARP, dtype=np.int64)
    base = first[order]
    rank = np.arange(WARP) - np.searchsorted(base, base, side="left")
    if (rank >= it).any():
        raise MappingError("more sub-vectors than lanes in an exchange group; use shared fusion")
    remap[order] = base + rank
    if np.unique(remap).size != WARP:
        raise MappingError("thread remap is not a bijection over the warp")
    return remap


def build_shuffle_schedule(layouts: LayoutPair, style: str = STYLE_STRIDED) -> ShuffleSchedule:
    tile = default_warp_tile(layouts, style)
    remap = build_thread_mapping(tile, layouts)
    it = layouts.iters
    return ShuffleSchedule(layouts, tile, it, tuple(int(x) for x in remap), tuple(range(1, it)))


def dequant_register_file(schedule: ShuffleSchedule) -> np.ndarray:
    """(32, iters, dst) element ids each lane holds right after dequantization."""
    src, dst, it = schedule.layouts.layout_src, schedule.layouts.layout_dst, schedule.layouts.iters
    elems = schedule.subvector_of_lane[:, None] * src + np.arange(src)
    return elems.reshape(WARP, it, dst)


def run_shuffle_steps(schedule: ShuffleSchedule, regs: np.ndarray) -> np.ndarray:
    """Warp-synchronous xor exchanges: at step ``off`` lane l receives its partner's
    (l ^ off) slot (l mod iters) into its own slot (partner mod iters)."""
    it = schedule.mini_warp_size
    lane = np.arange(WARP)
    cur = np.array(regs, copy=True)
    for off in schedule.offsets:
        partner = lane ^ off
        cur[lane, partner % it] = cur[partner, lane % it].copy()
    return cur


def expected_compute_ownership(schedule: ShuffleSchedule) -> np.ndarray:
    tile, dst, it = schedule.tile, schedule.layouts.layout_dst, schedule.layouts.iters
    e = np.arange(tile.n_elements)
    lane, slot = compute_owner(tile, dst, e)
    key = lane * it + slot
    order = np.lexsort((e, key))
    return e[order].reshape(WARP, it, dst)
