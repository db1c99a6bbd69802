"""bench.py's multi-rank path end to end on one GPU: 2 or 4 ranks under torchrun share the
device (KVR_BENCH_BACKEND=gloo stages the collectives through host copies).  Checks
the contract line: whole-job value over both ranks, max-over-ranks time, the summary
reduce with the packed-trace checksum, and e2e aggregated over ranks; and, for the
default config-5 workload (one fixed trial list sharded by (t div 2) mod N), that every
trial's result bytes at N ranks equal the 1-rank run (P20)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("N", [2, 4])
def test_bench_ranks_one_gpu(N):
    env = dict(os.environ, KVR_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(N),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", str(N),
           "--workload", "c2", "--steps", "2", "--warmup", "3", "--queries", "3000", "--trials", "64",
           "--no-cpu-baseline"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == N and d["trial_status_nonzero"] == 0
    rs = d["reduced_summary"]
    assert rs["trials"] == 64 * N and rs["queries"] == 64 * N * 3000
    assert rs["trace_hash_consistent"] is True and rs["status_nonzero"] == 0
    # value = both ranks' query-replays over the slowest rank's time
    assert abs(d["value"] - 64 * N * 3000 / (d["ms_per_step"] / 1e3)) <= 1e-6 * d["value"]
    e = d["e2e"]
    assert abs(e["value"] - e["queries_per_step"] / (e["ms_per_step"] / 1e3)) <= 1e-6 * e["value"]
    assert e["queries_per_step"] == 64 * N * 3000


def _c5(N, dump, trials):
    env = dict(os.environ, KVR_BENCH_BACKEND="gloo")
    if N == 1:
        cmd = [sys.executable, "bench.py"]
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(N),
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py"]
    cmd += ["--gpus", str(N), "--steps", "1", "--warmup", "3", "--trials", str(trials),
            "--no-cpu-baseline", "--dump-results", dump]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_c5_sharding_invariance(tmp_path):
    """P20: the config-5 list (480 trials over the 48 cells) run on 1 rank and on 3 ranks
    (one GPU, gloo): per-trial kvr_trial_result bytes identical, every trial exactly once."""
    import numpy as np
    trials = 480
    d1 = _c5(1, str(tmp_path / "n1"), trials)
    d3 = _c5(3, str(tmp_path / "n3"), trials)
    assert d1["scaling"] == d3["scaling"] == "strong"
    assert d1["trial_status_nonzero"] == 0 and d3["trial_status_nonzero"] == 0
    assert d3["reduced_summary"]["trials"] == trials
    assert d3["reduced_summary"]["trace_hash_consistent"] is True

    def load(prefix, ranks):
        tids, res = [], []
        for r in range(ranks):
            z = np.load(f"{prefix}.rank{r}.npz")
            tids.append(z["tids"])
            res.append(z["results"].reshape(len(z["tids"]), 144))
        tids, res = np.concatenate(tids), np.concatenate(res)
        order = np.argsort(tids)
        return tids[order], res[order]

    t1, r1 = load(str(tmp_path / "n1"), 1)
    t3, r3 = load(str(tmp_path / "n3"), 3)
    assert np.array_equal(t1, np.arange(trials)) and np.array_equal(t3, t1)
    assert np.array_equal(r1, r3)
