"""The bench's correctness gate and its N>1 path (BASELINE config 5) on the
GPU: the all-reduced checksum of one region pass over regenerated inputs
must equal the oracle's whole-range checksum at every rank count."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _last_json(out):
    for line in reversed(out.splitlines()):
        line = line.strip()
        if line.startswith("{"):
            return json.loads(line)
    raise AssertionError("no JSON line in:\n" + out)


def _bench(extra, nproc=1, env_extra=None, timeout=600):
    env = dict(os.environ)
    env.update(env_extra or {})
    base = ["bench.py", "--steps", "3", "--warmup", "3", "--only-stream", "--no-e2e",
            "--no-cpu"] + extra
    if nproc == 1:
        cmd = [sys.executable] + base
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={nproc}", "--master-addr", "127.0.0.1",
               "--master-port", str(_free_port())] + base + ["--gpus", str(nproc)]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return _last_json(r.stdout)


def test_bench_gate_fixture_size():
    """N=1, a size the committed fixture lists (2^22): checksum_ok."""
    d = _bench(["--elements", str(1 << 22)])
    assert d["checksum_ok"] is True
    assert d["correctness_gate"]["expected_from"].startswith("tests/golden")
    assert d["n_gpus"] == 1 and d["scaling"] == "strong"
    assert d["wall_window"]["ms"] > 0 and d["per_gpu_GBps"][0] > 0


def test_bench_gate_oracle_size():
    """N=1, a ragged size the fixture does not list: the oracle checker."""
    d = _bench(["--elements", "3000001"])
    assert d["checksum_ok"] is True
    assert "oracle" in d["correctness_gate"]["expected_from"]


@pytest.mark.parametrize("nproc,scaling", [(2, "strong"), (3, "weak")])
def test_bench_multi_rank_gate_on_one_gpu(nproc, scaling):
    """The torchrun path (sharding, both clocks, checksum all-reduce, one
    line from rank 0) with every rank on cuda:0 over gloo: the gathered
    checksum equals the whole range's.  Its throughput means nothing; the
    wall window shows the ranks shared one GPU."""
    n = (1 << 22) + 7 if scaling == "strong" else 1 << 21
    d = _bench(["--elements", str(n), "--scaling", scaling], nproc=nproc,
               env_extra={"OMPDS_BENCH_SHARE_GPU": "1", "OMPDS_BENCH_BACKEND": "gloo"})
    assert d["checksum_ok"] is True, d["correctness_gate"]
    assert d["n_gpus"] == nproc and len(d["per_gpu_GBps"]) == nproc
    total = n if scaling == "strong" else n * nproc
    assert d["config"]["elements_total"] == total
