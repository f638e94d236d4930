"""Seeded synthetic inputs (shared by oracle side and product side; holds no method arithmetic)."""
from . import rng, configs  # noqa: F401
