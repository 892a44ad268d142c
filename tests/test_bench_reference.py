"""bench.py --impl reference (the oracle arm) on CPU: one JSON line from rank 0
under torchrun with two ranks, the other rank exiting 0 without work, the
oracle using every host core despite torchrun's OMP_NUM_THREADS=1."""
import json
import os
import socket
import subprocess
import sys

from conftest import ROOT


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_reference_arm_torchrun_two_ranks():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           "bench.py", "--impl", "reference", "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--config", "cjm9_1024", "--ref-seconds", "0.3"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["working_ranks"] == 1
    assert d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["config"]["workload"] == "cjm9_1024"
    assert d["cpu_baseline"]["kind"] == "oracle"
    assert d["cpu_baseline"]["cores"] == len(os.sched_getaffinity(0))
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    # the measured step time (not a constant) and the GPU arm's config object
    sys.path.insert(0, ROOT)
    import bench
    assert d["config"] == bench.config_dict("cjm9_1024", 2)
    assert d["scaling"] == "strong"
    k = int(d["cpu_baseline"]["sample"].split()[0])
    assert abs(d["ms_per_step"] / 1e3 - k * 1024 * 1024 / (d["value"] * 1e9)) < 0.5 * d["ms_per_step"] / 1e3
    assert d["cpu_baseline"]["time_to_tol_extrapolated_s"] > 0
