"""B200-native butterfly merge (IOTA data-parallel merge step, arXiv 2507.17766).

``butterfly``  drop-in for iota_sim.butterfly (plan_shards, run_all_reduce, agreement, ...)
``device``     device-resident merge: DevicePlan (GPU index map), ButterflyMerge, Corruption
``simkernel``  BlobStore meter + RngStream used by the merge path
"""

from . import _lib, errors  # noqa: F401

__version__ = "0.1.0"
