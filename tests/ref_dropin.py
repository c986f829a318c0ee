"""pytest plugin (``-p ref_dropin``): run the reference's OWN tests, unmodified, against
the drop-in — the substitution INTEGRATION.md §2 / §4 describes.

* the attribute patch a maintainer appends to iota_sim/butterfly.py:
  ``plan_shards``, ``agreement``, ``mean_reducer`` and ``run_all_reduce`` of the
  reference module become the B200 ones, so the orchestrator and CLI (which look them
  up as ``butterfly.<attr>``, orchestrator.py:14,545-571) merge on the GPU;
* with BFLY_REF_SUBSTITUTE=module (default) the whole module is also replaced in
  ``sys.modules`` before collection, so ``from iota_sim.butterfly import ...`` in
  tests/test_butterfly.py:5-14 binds every name (pairs, plans, agreement, merge,
  analytics, types) to paper_2507_17766_b200.butterfly.

The reference itself comes from the git-ignored baseline/_ref (test infrastructure).
"""

import os
import sys

import iota_sim
import iota_sim.butterfly as _ref_butterfly

from paper_2507_17766_b200 import butterfly as _b200

for _name in ("plan_shards", "agreement", "mean_reducer", "run_all_reduce"):
    setattr(_ref_butterfly, _name, getattr(_b200, _name))

if os.environ.get("BFLY_REF_SUBSTITUTE", "module") == "module":
    sys.modules["iota_sim.butterfly"] = _b200
    iota_sim.butterfly = _b200
