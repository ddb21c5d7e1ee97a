"""bench.py's driver contract on CPU: the reference arm's JSON line (it runs
the compiled reference executor on host cores), the rank rule under a
multi-rank launch, and the warm-up floor.  The GPU arm is exercised by the
driver on a B200."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config")


def _reference_built():
    from oracle.oracle import Reference
    return Reference.available()


def _run(args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                          capture_output=True, text=True, timeout=600, env=e)


@pytest.mark.skipif(not _reference_built(), reason="oracle/_ref not built")
@pytest.mark.parametrize("cfg", (5, 2))
def test_reference_arm_json_line(cfg):
    r = _run(["--impl", "reference", "--config", str(cfg), "--size", "12", "--steps", "2",
              "--warmup", "3"])
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in KEYS:
        assert k in d, k
    assert d["impl"] == "reference"
    assert d["steps"] == 2 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["value"] > 0 and d["unit"] == "execs/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"]


def test_reference_arm_other_ranks_exit_silently():
    r = _run(["--impl", "reference", "--gpus", "2", "--size", "12", "--steps", "2", "--warmup", "3"],
             env={"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == ""


def test_gpus_must_match_world_size():
    r = _run(["--impl", "reference", "--gpus", "4", "--size", "12", "--steps", "2", "--warmup", "3"],
             env={"RANK": "0", "WORLD_SIZE": "2", "LOCAL_RANK": "0"})
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr


@pytest.mark.skipif(not _reference_built(), reason="oracle/_ref not built")
def test_gpus_flag_spawns_its_ranks():
    """--gpus 2 without torchrun: bench.py launches its two ranks itself
    (torch.distributed.run on 127.0.0.1); exactly one JSON line comes back."""
    env = {k: "" for k in ()}
    e = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--gpus", "2", "--size", "10", "--steps", "2", "--warmup", "3"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600, env=e)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference"
    assert d["config"]["global_systems"] == 8  # BASELINE's batch, whatever N


@pytest.mark.skipif(not _reference_built(), reason="oracle/_ref not built")
def test_reference_arm_matches_our_config_and_skips_the_package():
    r = _run(["--impl", "reference", "--config", "5", "--size", "10", "--steps", "2",
              "--warmup", "3"])
    assert r.returncode == 0, r.stderr
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["package_loaded"] is False
    import bench
    assert d["config"]["workload"] == bench.CONFIG_NAME[5]
    assert d["config"]["combo"] == 8 and d["config"]["global_systems"] == bench.GLOBAL_BATCH
    # the same object, key by key, as our arm prints for this workload
    n = 10 ** 3
    ours = bench.workload_config(5, 8, n, d["config"]["nnz_A"], d["config"]["nnz_L"],
                                 bench.GLOBAL_BATCH, 1)
    assert d["config"] == ours


def test_warmup_floor():
    r = _run(["--warmup", "2"])
    assert r.returncode != 0
    assert "warmup" in r.stderr
