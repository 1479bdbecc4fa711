"""bench.py's reference arm runs on the host alone (the reference CPU solver
from oracle/_ref, threads as ranks), so its JSON line — the one the driver
pairs with the GPU arm — is checked here without a GPU."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libcavity_ref.so")),
                    reason="reference library not built")
def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "1", "--cpu-seconds", "1"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["unit"] == "MCUPS" and line["higher_is_better"] is True
    assert line["metric"].startswith("cell-updates/s (MCUPS)")
    assert line["config"]["grid"] == [256, 256, 256] and line["dtype"] == "f64"
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == line["value"] > 0
    assert line["e2e"] == {"value": line["value"], "unit": "MCUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libcavity_ref.so")),
                    reason="reference library not built")
def test_reference_arm_never_loads_our_library():
    """The reference arm must run the reference alone: after it ran, the
    process has mapped oracle/_ref/libcavity_ref.so and not libcavity_b200.so."""
    code = ("import sys, json; sys.argv=['bench.py','--impl','reference','--gpus','2','--steps','2',"
            "'--warmup','1','--cpu-seconds','0.5']; sys.path.insert(0, %r); import bench; bench.main(); "
            "maps=open('/proc/self/maps').read(); "
            "print(json.dumps({'ref': 'libcavity_ref.so' in maps, 'ours': 'libcavity_b200' in maps}))" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = out.stdout.strip().splitlines()
    bench_line, maps = json.loads(lines[-2]), json.loads(lines[-1])
    assert maps == {"ref": True, "ours": False}
    # N=2 weak: the reference's own grow_grid gives the workload; config keys match our arm's
    assert bench_line["config"]["grid"] == [256, 256, 512]
    assert set(bench_line["config"]) == {"workload", "grid", "mode", "strategy", "overlap", "physics",
                                         "norm_history", "l2"}
    d = bench_line["decomposition"]
    assert d["np"] == bench_line["cpu_baseline"]["cores"] and d["timed_iterations"] == d["iterations"] - 1


def test_spawn_launcher_sets_torchrun_env(capfd):
    """`bench.py --gpus N` without torchrun spawns N workers with RANK,
    LOCAL_RANK, WORLD_SIZE and MASTER_* set, so they rendezvous over gloo."""
    sys.path.insert(0, ROOT)
    import bench
    code = ("import os, torch, torch.distributed as d; d.init_process_group('gloo'); "
            "t = torch.tensor([float(os.environ['LOCAL_RANK']) + 1]); d.all_reduce(t); "
            "print(os.environ['RANK'], os.environ['WORLD_SIZE'], int(t.item()), flush=True) "
            "if d.get_rank() == 0 else None; d.destroy_process_group()")
    rc = bench.spawn_ranks(3, [sys.executable, "-c", code])
    assert rc == 0
    assert capfd.readouterr().out.strip().splitlines()[-1] == "0 3 6"
