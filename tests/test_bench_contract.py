"""bench.py on the CPU: the reference arm's JSON line carries every key the
driver contract requires and describes the same workload as the GPU arm
(identical config block, same records by checksum), and the N-rank harness
(strong sharding, per-rank times, max-over-ranks) runs under torchrun with
gloo (--dry-run: no kernels).  The GPU arm itself is exercised on the B200."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from tests import _util as U

sys.path.insert(0, U.ROOT)
import bench  # noqa: E402


def _json_line(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out[-2000:]
    return json.loads(lines[0])


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(U.ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "1", "--records", "65536"], capture_output=True, text=True,
                       timeout=600, cwd=U.ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _json_line(r.stdout)
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["steps"] == 1 and d["n_gpus"] == 1 and d["vs_baseline"] is None and d["scaling"] == "strong"
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["kind"] == "reference" and cb["cores"] >= 1
    assert cb["sample"] and cb["unit"] == d["unit"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0
    # same workload description as the GPU arm, and the records it names
    cfg = dict(d["config"])
    cks = cfg.pop("input_checksum")
    assert cfg == bench.config_block(65536, 1)
    a = bench.host_corpus(3, 65536, bench.SEED)
    assert cks == f"{bench.checksum_u64(a):016x}"


def test_host_corpus_is_counter_based_and_sharded_consistently():
    whole = bench.host_corpus(5, 5000, 7, first=(1 << 20) - 2500, threads=3)
    part = bench.host_corpus(5, 2500, 7, first=1 << 20, threads=1)
    assert (whole[2500:].view(np.uint64) == part.view(np.uint64)).all()
    for cfg in (1, 2, 3, 4):
        a = bench.host_corpus(cfg, 4096, 11)
        assert np.isfinite(a).all()
    sym = bench.host_corpus(1, 4096, 11).reshape(-1, 3, 3)
    assert (sym == sym.transpose(0, 2, 1)).all()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_torchrun_strong_sharding_dry_run(world):
    n = 1000001
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                        "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
                        os.path.join(U.ROOT, "bench.py"), "--dry-run", "--gpus", str(world), "--records", str(n),
                        "--steps", "3", "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=U.ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _json_line(r.stdout)
    assert d["n_gpus"] == world and d["scaling"] == "strong"
    assert len(d["per_rank_ms"]) == world
    assert d["ms_per_step"] == pytest.approx(max(d["per_rank_ms"]) / 3)
    shards = d["shards"]
    assert shards[0][0] == 0 and shards[-1][1] == n
    assert all(b[0] == a[1] for a, b in zip(shards, shards[1:]))
    assert d["config"]["records_per_gpu"] == [hi - lo for lo, hi in shards]
    assert d["rank_objects"] == list(range(1, world + 1))  # all_gather_object over the gloo group
    assert sum(d["config"]["records_per_gpu"]) == n == d["config"]["records_total"]
