"""Synthetic input production for the tests and the benchmark.

Not the product and not the checker: the reference's corpus generator
(fdata.py:170-347) restated so the corpora here are the same bytes as the
reference's, which the golden fixtures and the parity tests depend on.
SURVEY.md §2 marks host-side input generation out of scope for the hot path;
the product's on-device plane generator (csrc/synth.cu) consumes the
per-node base images this module produces.
"""

from .synth import SyntheticCorpus, gen_synthetic, gen_synthetic_device, synth_base

__all__ = ["SyntheticCorpus", "gen_synthetic", "gen_synthetic_device", "synth_base"]
