"""bench.py launcher and reference-arm hygiene (CPU only)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _last_json(out):
    return json.loads([l for l in out.splitlines() if l.startswith("{")][-1])


def test_gpus_2_reaches_two_ranks():
    """`python bench.py --gpus 2` without torchrun re-launches itself under
    torch.distributed.run with 2 processes (the driver's N > 1 form)."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    d = _last_json(r.stdout)
    assert d["world_size"] == 2 and d["ranks_reached"] == 2


def test_reference_arm_loads_only_the_oracle():
    """The reference arm builds its instance with the oracle's own generator
    and config: the only in-tree library in the process is oracle/."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload",
                        "ladybug-49", "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr
    d = _last_json(r.stdout)
    assert d["impl"] == "reference" and d["repo_libs_loaded"] == ["oracle/liboracle_dba.so"]
    assert d["config"]["workload"] == "ladybug-49" and d["value"] > 0
    cb = d["cpu_baseline"]
    assert cb["cores"] >= 1 and cb["k1"]["cores"] == 1 and cb["detail"]["full_pcg_iterations"] > 0
    assert "paper_2112_01349_b200" not in r.stderr
