"""Hierarchical fusion planning (vqforge.fusion, pkg/src/vqforge/fusion.py; paper §VI-B, Alg. 1).

The planner decides whether dequantized data reaches the compute layout through
intra-warp register exchanges (``n_shuffle = v / required_layout - 1`` xor
steps inside mini-warps) or through shared memory, using the profiled latency
ratio THRES_SHUFFLE.

How the B200 kernels realise the two levels:
* "register": GEMV and decode attention are CUDA-core kernels where each lane
  owns whole sub-vectors and consumes them itself with fma.rn.f32.f16 — the
  exchange schedule degenerates to zero shuffles.
* "shared": tcgen05.mma reads operands only from shared memory / TMEM, so the
  prefill GEMM always stages dequantized tiles in shared memory in the UMMA
  canonical layout.
The schedule construction below is kept for API parity and is verified against
the reference's exhaustive ownership oracle in tests.
"""

import json
from dataclasses import dataclass

import numpy as np

from .errors import MappingError

WARP = 32
THRES_SHUFFLE = 5
STYLE_STRIDED = "strided"
STYLE_MMA = "mma"


def _pow2(n: int) -> bool:
    return n > 0 and not n & (n - 1)


@dataclass(frozen=True)
class LayoutPair:
    layout_src: int
    layout_dst: int

    def __post_init__(self):
        if not (_pow2(self.layout_src) and _pow2(self.layout_dst)):
            raise MappingError(f"layouts must be powers of two, got {self.layout_src}/{self.layout_dst}")

    @property
    def register_compatible(self) -> bool:
        return self.layout_src >= self.layout_dst

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
    if layouts.register_compatible and layouts.n_shuffle < thres_shuffle:
        return "register"
    return "shared"


@dataclass(frozen=True)
class WarpTile:
    rows: int
    cols: int
    style: str

    @property
    def n_elements(self) -> int:
        return self.rows * self.cols


def default_warp_tile(layouts: LayoutPair, style: str) -> WarpTile:
    src = layouts.layout_src
    if style == STYLE_STRIDED:
        return WarpTile(WARP, src, style)
    if style == STYLE_MMA:
        if layouts.layout_dst != 2:
            raise MappingError("mma consumers take layout_dst = 2")
        return WarpTile(WARP, src, STYLE_STRIDED) if src < 4 else WarpTile(16, 2 * src, style)
    raise MappingError(f"unknown compute style {style!r}")


def compute_owner(tile: WarpTile, dst: int, e: np.ndarray):
    """(lane, slot) consuming element e in the compute layout."""
    if tile.style == STYLE_STRIDED:
        return (e // dst) % WARP, e // (WARP * dst)
    r, c = np.divmod(e, tile.cols)
    return (r % 8) * 4 + (c % 8) // 2, (r // 8) * (tile.cols // 8) + c // 8


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
        inv = np.empty(WARP, dtype=np.int64)
        inv[np.asarray(self.thread_remap)] = np.arange(WARP)
        return inv

    def to_json(self) -> str:
        return json.dumps({"mini_warp_size": self.mini_warp_size, "remap": list(self.thread_remap),
                           "offsets": list(self.offsets)})


def build_thread_mapping(warp_tile: WarpTile, layouts: LayoutPair) -> np.ndarray:
    """remap[naive dequant lane] = lane that dequantizes it, so every mini-warp of
    ``iters`` lanes dequantizes exactly what it consumes (Alg. 1 lines 2-11)."""
    src, dst, it = layouts.layout_src, layouts.layout_dst, layouts.iters
    if it > WARP:
        raise MappingError(f"exchange group of {it} lanes exceeds the warp; use shared fusion")
    e = np.arange(warp_tile.n_elements)
    consumer, _ = compute_owner(warp_tile, dst, e)
    producer = e // src
    groups = {}
    for lane in range(WARP):
        key = tuple(dict.fromkeys(consumer[producer == lane].tolist()))
        groups.setdefault(key, []).append(lane)
    remap = np.full(WARP, -1, dtype=np.int64)
    for key, lanes in groups.items():
        if len(key) != it or len(lanes) != it:
            raise MappingError(f"consumer set {key} of lanes {lanes} is not an {it}-lane exchange "
                               "group; use shared fusion")
        if key[0] % it or key != tuple(range(key[0], key[0] + it)):
            raise MappingError(f"consumer set {key} is not xor-aligned; use shared fusion")
        remap[sorted(lanes)] = key
    if (remap < 0).any() or np.unique(remap).size != WARP:
        raise MappingError("thread remap is not a bijection over the warp")
    return remap


def build_shuffle_schedule(layouts: LayoutPair, style: str = STYLE_STRIDED) -> ShuffleSchedule:
    tile = default_warp_tile(layouts, style)
    remap = build_thread_mapping(tile, layouts)
    it = layouts.iters
    return ShuffleSchedule(layouts, tile, it, tuple(int(x) for x in remap), tuple(range(1, it)))


def dequant_register_file(schedule: ShuffleSchedule) -> np.ndarray:
    """(32, iters, dst) element ids right after dequantization under the remap."""
    src, dst, it = schedule.layouts.layout_src, schedule.layouts.layout_dst, schedule.layouts.iters
    sub = schedule.subvector_of_lane
    return (sub[:, None] * src + np.arange(src)[None, :]).reshape(WARP, it, dst)


def run_shuffle_steps(schedule: ShuffleSchedule, regs: np.ndarray) -> np.ndarray:
    """Warp-synchronous xor exchanges: step ``off`` swaps slot (lane^off) % iters with lane^off."""
    it = schedule.mini_warp_size
    lanes = np.arange(WARP)
    cur = regs.copy()
    for off in schedule.offsets:
        partner = lanes ^ off
        prev = cur.copy()
        cur[lanes, partner % it] = prev[partner, lanes % it]
    return cur


def expected_compute_ownership(schedule: ShuffleSchedule) -> np.ndarray:
    tile, dst, it = schedule.tile, schedule.layouts.layout_dst, schedule.layouts.iters
    e = np.arange(tile.n_elements)
    lane, slot = compute_owner(tile, dst, e)
    want = np.empty((WARP, it, dst), dtype=np.int64)
    for ln in range(WARP):
        for j in range(it):
            want[ln, j] = np.sort(e[(lane == ln) & (slot == j)])
    return want
