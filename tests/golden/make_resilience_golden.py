"""Fixture for the resilience Monte-Carlo, from the REFERENCE's own
butterfly.monte_carlo_resilience (read-only /root/reference, butterfly.py:322-341).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_resilience_golden.py
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
from iota_sim import butterfly as b  # noqa: E402

out = {}
for n, ks, trials, seed in [(50, [0, 1, 2, 5, 10, 25, 50], 1000, 2), (8, [0, 2, 3, 8], 37, 5), (2, [0, 1, 2], 3, 0),
                            (130, [7, 64], 11, 9)]:
    r = b.monte_carlo_resilience(n, ks, trials, seed)
    out[f"{n}_{trials}_{seed}"] = {str(k): v for k, v in r.items()}
(Path(__file__).resolve().parent / "resilience_mc.json").write_text(json.dumps(out))
