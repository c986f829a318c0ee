"""Run one iota-sim CLI scenario (``train``) and write its CSVs to OUT.

    python tests/_ref_scenario.py CONFIG OUT [b200]

With ``b200`` the reference's butterfly module is patched as INTEGRATION.md §2 shows
(the merges of every layer and stage run through paper_2507_17766_b200), otherwise the
reference runs as shipped.  Used by tests/test_reference_suite.py to compare the two
runs' CSVs byte for byte.
"""

import sys

import iota_sim.butterfly as ref_butterfly
from iota_sim.cli import main

if len(sys.argv) > 3 and sys.argv[3] == "b200":
    from paper_2507_17766_b200 import butterfly as b200

    for name in ("plan_shards", "agreement", "mean_reducer", "run_all_reduce"):
        setattr(ref_butterfly, name, getattr(b200, name))
    calls = {"n": 0}
    real = b200.run_all_reduce

    def counted(*a, **k):
        calls["n"] += 1
        return real(*a, **k)

    ref_butterfly.run_all_reduce = counted
    try:
        main(["train", "--config", sys.argv[1], "--out", sys.argv[2]], standalone_mode=False)
    finally:
        print("B200_MERGES", calls["n"])
else:
    main(["train", "--config", sys.argv[1], "--out", sys.argv[2]], standalone_mode=False)
