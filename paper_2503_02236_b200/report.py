"""Counters returned with every fused launch (vqforge.report, pkg/src/vqforge/report.py:22-89).

The reference *simulates* these counters. On B200 the executor fills them from
the launch plan's algorithmic traffic (what the kernel must move), and puts the
measured quantities — kernel name, microseconds, achieved GB/s — in ``meta``.
Schema version 1 and the CSV columns are unchanged so existing tooling reads them.
"""

import csv
import json
from dataclasses import asdict, dataclass, field

SCHEMA_VERSION = 1
COUNTERS = ("bank_conflicts", "global_to_shared_bytes", "shared_to_reg_bytes",
            "staged_dequant_bytes", "global_bytes", "reduce_bytes", "occupancy",
            "quant_invocations")
CSV_COLUMNS = ["variant", *COUNTERS]


@dataclass
class SimReport:
    bank_conflicts: int = 0
    global_to_shared_bytes: int = 0
    shared_to_reg_bytes: int = 0
    staged_dequant_bytes: int = 0
    global_bytes: int = 0
    reduce_bytes: int = 0
    occupancy: int = 0
    quant_invocations: int = 0
    meta: dict = field(default_factory=dict)

    def merge(self, other: "SimReport") -> "SimReport":
        """Counter-wise sum; occupancy is per launch and kept from ``self``."""
        merged = {k: getattr(self, k) + getattr(other, k) for k in COUNTERS if k != "occupancy"}
        return SimReport(occupancy=self.occupancy or other.occupancy, meta=dict(self.meta), **merged)

    def validate(self) -> None:
        for k in COUNTERS:
            if getattr(self, k) < 0:
                raise ValueError(f"counter {k} went negative")

    def to_dict(self) -> dict:
        d = asdict(self)
        d["schema_version"] = SCHEMA_VERSION
        return d

    def to_json(self, **kw) -> str:
        return json.dumps(self.to_dict(), **kw)


def write_reports_csv(rows, path) -> None:
    """rows: iterable of (variant name, SimReport)."""
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(CSV_COLUMNS)
        for name, rep in rows:
            w.writerow([name, *(getattr(rep, k) for k in COUNTERS)])
