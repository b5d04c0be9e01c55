"""Evaluation record (mirrors lshclust.metrics, metrics.py:1-59).

`MetricsRecord` carries the reference's nine fields with the same JSON
encoding (sorted keys, non-finite summaries rejected), so records from the
two implementations compare field by field.  One extension, `device`, holds
what the B200 run adds -- points/s, per-phase roofline fractions, the
assignment recheck counts and the rank-split boundary exceptions; it is
omitted from the JSON when empty, so a record without it is byte-compatible
with the reference's.
"""

from __future__ import annotations

import json
import math
from dataclasses import asdict, dataclass, field

from .data import Clustering

__all__ = ["MetricsRecord", "evaluate", "device_summary"]


@dataclass
class MetricsRecord:
    k_star: int
    max_radius: float
    mean_radius: float
    objective: float
    radii: list
    sizes: list
    stage_seconds: dict = field(default_factory=dict)
    transport_bytes: dict = field(default_factory=dict)
    parameters: dict = field(default_factory=dict)
    device: dict = field(default_factory=dict)

    def to_json(self) -> str:
        d = asdict(self)
        for key in ("max_radius", "mean_radius", "objective"):
            if not math.isfinite(d[key]):
                raise ValueError(f"non-finite metric {key}")
        if not d["device"]:
            d.pop("device")
        return json.dumps(d, sort_keys=True)

    @classmethod
    def from_json(cls, text: str) -> "MetricsRecord":
        return cls(**json.loads(text))


def evaluate(clustering: Clustering, stage_seconds=None, transport_bytes=None, parameters=None,
             device=None) -> MetricsRecord:
    """k* (non-empty clusters), per-cluster radii, their max and size-weighted
    mean, and the assignment objective (metrics.py:41-59)."""
    sizes = clustering.sizes
    occupied = sizes > 0
    radii = clustering.radii[occupied]
    weights = sizes[occupied]
    mean_radius = float((radii * weights).sum() / weights.sum()) if weights.sum() else 0.0
    return MetricsRecord(
        k_star=clustering.k_star,
        max_radius=float(radii.max()) if radii.size else 0.0,
        mean_radius=mean_radius,
        objective=float(clustering.objective),
        radii=[float(r) for r in clustering.radii],
        sizes=[int(s) for s in sizes],
        stage_seconds=dict(stage_seconds or {}),
        transport_bytes=dict(transport_bytes or {}),
        parameters=dict(parameters or {}),
        device=dict(device or {}),
    )


# per-point algorithmic work of each phase; peaks: MEASURED_PEAKS.json
# values on B200 (HBM copy GB/s, dense bf16 TFLOP/s)
_HBM_GBS = 6536.7
_TENSOR_TFLOPS = 1601.3


def device_summary(result, n: int, d: int, tables: int, wall_seconds: float) -> dict:
    """The `device` extension of a pipeline run: end-to-end points/s, each
    phase's achieved rate as a fraction of its roofline (bucketize and SILK
    bytes against HBM, assignment flops against the tensor pipe), and the
    exactness counters (screen rechecks, full scans, rank-split boundary
    exceptions when the run computed them)."""
    t = result.timings
    info = getattr(result, "info", {}) or {}
    k = len(result.seed_groups) if n <= 10 ** 6 else result._groups.count
    phases = {}

    def frac(name, sec, work, peak, unit):
        if sec and sec > 0:
            ach = work / sec / (1e9 if unit == "GB/s" else 1e12)
            phases[name] = {"achieved": round(ach, 3), "unit": unit, "frac": round(ach / peak, 5)}

    frac("bucketize", t.get("transform", 0) + t.get("sync_buckets", 0), n * (4 * d + 4 * tables), _HBM_GBS, "GB/s")
    frac("seeding", t.get("seeding", 0), n * 4 * tables, _HBM_GBS, "GB/s")
    if d:
        frac("assign", t.get("assign", 0), 2.0 * n * k * d, _TENSOR_TFLOPS, "TFLOP/s")
    out = {"points_per_sec": n / wall_seconds if wall_seconds > 0 else None, "phases": phases}
    for key in ("assign_rechecked", "assign_full_scans"):
        if key in info:
            out[key] = info[key]
    sb = info.get("split_boundary")
    if sb is not None:
        out["split_boundary"] = {"ambiguous": sb["ambiguous"], "within_rel": sb["within_rel"]}
    return out
