"""The reference's OWN hot-path tests, unmodified, through the drop-in.

The reference (iota-sim, git-ignored baseline/_ref, installed by __graft_entry__.build()
with the base contract's pip command; its tests copied beside it) is run in a
subprocess with the ``ref_dropin`` plugin, which applies the substitution of
INTEGRATION.md §2/§4.  Nothing here reads /root/reference.

* CPU: the tests of pkg/tests/test_butterfly.py that need no device (pairs, plans,
  the seed-24 KAT, the chi-square uniformity, analytics, the ShapeError of agreement)
  — the exception classes raised by the drop-in must be iota_sim's;
* GPU: all 22 tests of test_butterfly.py and acceptance criteria 1, 2, 3, 4 and 9
  (pkg/tests/test_acceptance.py:43-162,326-352);
* GPU: a 3-epoch orchestrator scenario with deceptive and lazy miners and compressed
  sharing stages through the CLI (orchestrator.py:519-606, cli.py:85-136): every CSV
  byte-identical with the drop-in patched in and with the reference as shipped;
* GPU: the reference's whole shipped suite (158 tests) with the attribute patch.
"""

import hashlib
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"
REF_TESTS = REF / "tests"

needs_ref = pytest.mark.skipif(not (REF / "iota_sim").is_dir() or not REF_TESTS.is_dir(),
                               reason="baseline/_ref (the reference) is not installed; run __graft_entry__.build()")


def _env(mode="module"):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT), str(ROOT / "tests"), str(REF)])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    env["BFLY_REF_SUBSTITUTE"] = mode
    return env


def _pytest(args, mode="module", timeout=900):
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p", "ref_dropin",
           "--rootdir", str(REF_TESTS), *args]
    r = subprocess.run(cmd, cwd=str(REF_TESTS), env=_env(mode), capture_output=True, text=True, timeout=timeout)
    return r.returncode, r.stdout + r.stderr


CPU_SELECTION = "TestPairs or TestShardPlan or TestResilience or test_shape_mismatch"


@needs_ref
def test_reference_butterfly_tests_cpu_subset():
    rc, out = _pytest(["test_butterfly.py", "-k", CPU_SELECTION])
    assert rc == 0, out
    assert "15 passed" in out, out


@needs_ref
def test_plugin_substitutes_the_module():
    code = ("import ref_dropin, iota_sim, iota_sim.butterfly as b, iota_sim.errors as e; "
            "import paper_2507_17766_b200.butterfly as ours, paper_2507_17766_b200.errors as oe; "
            "assert b is ours and oe.ShapeError is e.ShapeError and ours.ShardPlan.__module__ == 'iota_sim.butterfly'; "
            "print('ok')")
    r = subprocess.run([sys.executable, "-c", code], env=_env(), capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
@needs_ref
def test_reference_butterfly_tests_all(cuda_device):
    rc, out = _pytest(["test_butterfly.py"])
    assert rc == 0, out
    assert "22 passed" in out, out


@pytest.mark.gpu
@needs_ref
def test_reference_acceptance_criteria(cuda_device):
    sel = "criterion_1 or criterion_2 or criterion_3 or criterion_4 or criterion_9"
    rc, out = _pytest(["test_acceptance.py", "-k", sel, "-s"], mode="attribute")
    assert rc == 0, out
    assert "5 passed" in out, out
    for c in ("criterion 1", "criterion 2", "criterion 3", "criterion 4", "criterion 9"):
        assert f"ACCEPTANCE {c}" in out and "FAIL" not in out, out


SCENARIO = """[train]
dims = [4, 16, 16, 2]
miners = [["honest", "lazy:0.3", "honest", "deceptive:1.5"], ["honest", "deceptive:2.0", "honest", "honest", "lazy:0.5"], ["honest", "honest", "deceptive:1.5"]]
seed = 9
epochs = 3
b_min = 2
trigger_fraction = 0.5
batch_size = 4
compressed_stages_per_epoch = 1
compression_ratio = 4.0
"""


@pytest.mark.gpu
@needs_ref
def test_orchestrator_scenario_csvs_byte_identical(cuda_device, tmp_path):
    cfg = tmp_path / "scenario.toml"
    cfg.write_text(SCENARIO)
    hashes = {}
    for arm in ("reference", "b200"):
        out = tmp_path / arm
        cmd = [sys.executable, str(ROOT / "tests" / "_ref_scenario.py"), str(cfg), str(out)]
        if arm == "b200":
            cmd.append("b200")
        r = subprocess.run(cmd, env=_env("attribute"), capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stdout + r.stderr
        if arm == "b200":
            merges = int(r.stdout.split("B200_MERGES")[1].split()[0])
            assert merges >= 12, r.stdout  # most (epoch, stage, layer) merges went through the drop-in
        hashes[arm] = {p.name: hashlib.sha256(p.read_bytes()).hexdigest() for p in sorted(out.glob("*.csv"))}
    assert len(hashes["reference"]) >= 6
    assert hashes["b200"] == hashes["reference"]


@pytest.mark.gpu
@needs_ref
def test_broadcastable_callable_outputs_match_reference(cuda_device):
    """A corruption callable returning a scalar: a lone survivor's scalar is
    broadcast into merged (numpy assignment, butterfly.py:263); two survivors whose outputs
    have different shapes raise ShapeError in agreement (:125-126); equal-shape scalars
    are compared and adopted.  The drop-in against the reference itself, in-process."""
    import numpy as np

    sys.path.append(str(REF))
    import iota_sim.butterfly as ref
    from iota_sim.errors import ShapeError as RefShapeError
    from iota_sim.simkernel import BlobStore as RefStore

    from paper_2507_17766_b200 import butterfly as bf

    def run(mod, n, P, seed, failures, corr):
        rng = np.random.default_rng(seed)
        payloads = {m: rng.uniform(-1, 1, P) for m in range(n)}
        plan = ref.plan_shards(ref.enumerate_pairs(n), P, 4, seed)
        store = RefStore()
        res = mod.run_all_reduce(store, payloads, plan, failures=frozenset(failures), corruptions=corr)
        meter = {a: (m.bytes_uploaded, m.bytes_downloaded) for a, m in store.meter.items()}
        return res, meter, {k: bytes(v) for k, v in store.objects.items()}

    cases = [
        (3, 31, 1, {0, 1}, {2: lambda red: np.float64(3.0)}),          # lone survivor: broadcast
        (2, 17, 2, set(), {0: lambda red: np.float64(5.0), 1: lambda red: np.float64(5.0)}),  # equal scalars
        (2, 17, 3, set(), {0: lambda red: np.full(1, 2.0), 1: lambda red: np.full(1, -2.0)}),  # (1,) copies disagree
    ]
    for n, P, seed, failures, corr in cases:
        want, wmeter, wobj = run(ref, n, P, seed, failures, corr)
        got, gmeter, gobj = run(bf, n, P, seed, failures, corr)
        assert np.array_equal(np.asarray(got.merged).view(np.uint64), np.asarray(want.merged).view(np.uint64))
        assert got.shard_status == want.shard_status and got.flagged == want.flagged
        assert np.array_equal(np.isnan(got.agreement_matrix.entries), np.isnan(want.agreement_matrix.entries))
        m = ~np.isnan(want.agreement_matrix.entries)
        assert np.allclose(got.agreement_matrix.entries[m], want.agreement_matrix.entries[m], rtol=0, atol=1e-12)
        assert gmeter == wmeter and gobj == wobj
    # different shapes on the two survivors: ShapeError from both (the reference's class)
    for mod in (ref, bf):
        with pytest.raises(RefShapeError):
            run(mod, 3, 31, 4, set(), {2: lambda red: np.float64(3.0)})


@pytest.mark.gpu
@needs_ref
def test_reference_whole_suite_through_dropin(cuda_device):
    """Every test file the reference ships (pkg/tests: butterfly, acceptance, orchestrator,
    CLI, validator, incentives, CLASP, simkernel, model, backends) — 158 tests — with the
    drop-in patched in by attribute, so every merge the orchestrator
    makes in those tests runs on the GPU."""
    rc, out = _pytest([], mode="attribute", timeout=1800)
    assert rc == 0, out[-6000:]
    assert "158 passed" in out, out[-3000:]
