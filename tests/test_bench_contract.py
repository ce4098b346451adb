"""bench.py contract checks that need no GPU: the reference arm (the CPU oracle, rank 0 only)
prints one JSON line with the keys the driver reads, non-zero ranks of a torchrun launch exit
0 without output, and the multi-rank partition plans (weak and strong scaling) under gloo."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None):
    env = dict(os.environ)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                          text=True, env=env, timeout=600)


def test_reference_arm_prints_one_json_line():
    r = _run(["--impl", "reference", "--steps", "1", "--warmup", "3"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("C3")  # the metric's configuration (configs[2])
    assert "2097152 DOFs" in d["config"]["sample"]  # the same 2^21-DOF slab as cpu_baseline


def test_reference_arm_nonzero_rank_is_silent():
    r = _run(["--impl", "reference", "--steps", "1", "--warmup", "3", "--gpus", "2"],
             {"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert r.returncode == 0, r.stderr[-2000:]
    assert not [l for l in r.stdout.splitlines() if l.startswith("{")]


def _torchrun(nproc, args):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + os.getpid() % 2000),
           os.path.join(ROOT, "bench.py"), *args]
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")  # CPU: gloo process group
    return subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600)


def _plan(r):
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 only
    return json.loads(lines[0])


def test_strong_scaling_plan_splits_the_fixed_global_grid():
    """--scaling strong (SURVEY §8(d) E(G) = t(1)/(G t(G))): the config's global grid is split into
    contiguous z-slabs whose sizes sum to the global N, with no gaps or overlaps."""
    for cfg, nz, G in (("c3", 512, 2), ("c2", 128, 3)):
        d = _plan(_torchrun(G, ["--same-gpu", "--gpus", str(G), "--scaling", "strong", "--config", cfg, "--dry-run"]))
        assert d["scaling"] == "strong" and d["n_gpus"] == G and d["nz_global"] == nz
        sl = sorted(d["slabs"], key=lambda s: s["rank"])
        assert [s["rank"] for s in sl] == list(range(G))
        assert sl[0]["z0"] == 0 and sl[-1]["z1"] == nz
        assert all(a["z1"] == b["z0"] for a, b in zip(sl, sl[1:]))
        assert sum(s["dofs"] for s in sl) == d["global_dofs"] == d["grid"][0] * d["grid"][1] * nz
        assert max(s["z1"] - s["z0"] for s in sl) - min(s["z1"] - s["z0"] for s in sl) <= 1


def test_weak_scaling_plan_gives_every_rank_a_full_slab():
    d = _plan(_torchrun(2, ["--same-gpu", "--gpus", "2", "--scaling", "weak", "--config", "c3", "--dry-run"]))
    assert d["scaling"] == "weak" and d["nz_global"] == 1024
    assert [s["dofs"] for s in d["slabs"]] == [512 * 512 * 512] * 2
