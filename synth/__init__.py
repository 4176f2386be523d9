"""Seeded synthetic inputs shared by the oracle tests and the product bench (no method arithmetic)."""
from .clouds import (CONFIG_NAMES, SEEDS, BATCH_SEED, Workload, make, make_batch, axis_angle,  # noqa: F401
                     random_rigid)
