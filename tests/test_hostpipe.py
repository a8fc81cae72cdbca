"""The host-buffer pipeline (paper_2511_00292_b200/csrc/eig33_host.cpp) on the
CPU: compiled against a mock CUDA runtime (tests/hostpipe/mock) whose
"kernels" are the product's per-record math built for the CPU, under
AddressSanitizer/UBSan and ThreadSanitizer.  Covers every host entry point
(direct and staged paths, ragged chunks, pinned and pageable buffers), the
multi-device shard driver (device lists, concurrent callers sharing the copy
pool), NotSymmetric's first-record index, error returns with injected launch
failures (no crash, no late writes, next call works) and restoration of the
caller's current device."""
import os
import subprocess

import pytest

from tests import _util as U

HP = os.path.join(U.ROOT, "tests", "hostpipe")
SRCS = [os.path.join(HP, "pipe_test.cpp"), os.path.join(HP, "mock_device.cpp"),
        os.path.join(U.ROOT, "paper_2511_00292_b200", "csrc", "eig33_host.cpp")]


def _build(tmp_path_factory, san):
    out = tmp_path_factory.mktemp("hostpipe") / f"pipe_test_{san}"
    flags = {"asan": ["-fsanitize=address,undefined", "-fno-sanitize-recover=undefined"],
             "tsan": ["-fsanitize=thread"]}[san]
    small = ["-DEIG33_HOST_CHUNK_LOG2=10", "-DEIG33_STAGE_CHUNK_LOG2=8", "-DEIG33_STAGE_MIN_BYTES=65536",
             "-DEIG33_COPY_PART=4096"]
    subprocess.run(["g++", "-O1", "-g", *flags, *small, "-std=c++17", "-pthread", "-mfma", "-ffp-contract=off",
                    "-I", os.path.join(HP, "mock"), "-o", str(out), *SRCS], check=True)
    return str(out)


@pytest.fixture(scope="module")
def asan(tmp_path_factory):
    return _build(tmp_path_factory, "asan")


@pytest.fixture(scope="module")
def tsan(tmp_path_factory):
    return _build(tmp_path_factory, "tsan")


def _run(exe, what, **env):
    e = dict(os.environ, MOCK_NDEV="2", **{k: str(v) for k, v in env.items()})
    r = subprocess.run([exe, what], capture_output=True, text=True, timeout=900, env=e)
    assert r.returncode == 0 and f"OK {what}" in r.stdout, (r.stdout + r.stderr)[-4000:]


@pytest.mark.parametrize("what", ["basic", "multi", "device"])
def test_host_pipeline_asan(asan, what):
    _run(asan, what)


@pytest.mark.parametrize("fail_at", [1, 2, 3, 6])
def test_host_pipeline_failed_launch_returns_cleanly(asan, fail_at):
    _run(asan, "fail", MOCK_FAIL_LAUNCH_AT=fail_at)


def test_host_pipeline_threads_tsan(tsan):
    _run(tsan, "multi", TSAN_OPTIONS="halt_on_error=1")
