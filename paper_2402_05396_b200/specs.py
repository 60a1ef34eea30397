"""Workload table of the five BASELINE.json shapes (A-E).

Dependency-free on purpose: bench.py's reference arm reads this table by
file path, so the reference's CPU timing never imports the product package
or maps its CUDA library.  ``shapes.py`` builds the device graphs.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class ShapeSpec:
    key: str
    name: str
    V: int
    E: int
    d_e: int
    d_v: int
    aggregator: str
    finder_policy: str
    adaptive: bool
    m: int
    n: int
    batch: int
    note: str = ""

    def config_fields(self, **over):
        """RunConfig fields (training.py:47-108) of this workload's hot path."""
        kw = dict(aggregator=self.aggregator, finder_policy=self.finder_policy, adaptive_neighbor=self.adaptive,
                  m=self.m, n=self.n, batch_size=self.batch, cache_fraction=0.2)
        if self.adaptive:
            kw["precision"] = "float32"  # the reference's fast mode (RunConfig.precision); tensor-core K7
        kw.update(over)
        return kw

    def path_config(self, **over):
        from .pipeline import PathConfig
        return PathConfig(**self.config_fields(**over))

    def scaled(self, factor):
        """Same node count and widths, E scaled (CPU-baseline samples)."""
        return ShapeSpec(self.key, self.name + f"/{factor:g}", self.V, max(1, int(self.E * factor)), self.d_e,
                         self.d_v, self.aggregator, self.finder_policy, self.adaptive, self.m, self.n, self.batch,
                         self.note)


SHAPES = {
    "A": ShapeSpec("A", "wikipedia", 9_227, 157_474, 172, 0, "graphmixer", "recent", False, 10, 10, 600,
                   "1-hop most-recent 10, batch 600"),
    "B": ShapeSpec("B", "reddit", 10_984, 672_447, 172, 0, "tgat", "uniform", False, 10, 10, 600,
                   "2-hop uniform 10x10, batch 600, 20% cache"),
    "C": ShapeSpec("C", "movielens", 10_000, 25_000_000, 266, 0, "graphmixer", "recent", True, 25, 10, 4000,
                   "adaptive 25->10 linear decoder, batch 4000; d_e 266 per PAPER.md:686"),
    "D": ShapeSpec("D", "flights", 13_169, 1_927_145, 172, 100, "tgat", "uniform", True, 25, 10, 600,
                   "2-hop adaptive 25->10 gatv2, 20% cache; d_v 100 (PAPER.md:685) + synthetic 172-d edges"),
    "E": ShapeSpec("E", "gdelt", 16_682, 191_290_882, 186, 0, "tgat", "recent", False, 10, 10, 600,
                   "2-hop most-recent 10x10, batch 600, 20% cache"),
}
