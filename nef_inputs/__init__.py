"""Seeded synthetic input generators (shared by the oracle and the CUDA path; holds
none of the method's arithmetic)."""
from .synth import CONFIGS, Config, factor_shapes, generate_numpy, generate_torch, split_labels  # noqa: F401
