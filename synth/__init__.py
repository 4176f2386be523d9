"""Seeded synthetic inputs shared by the oracle tests and the product bench (no method arithmetic)."""
from .clouds import CONFIG_NAMES, SEEDS, Workload, make, axis_angle, random_rigid  # noqa: F401
