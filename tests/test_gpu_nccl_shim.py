"""The NCCL transport of the partitioned optimize (csrc/partition.cu) at
world > 1 -- on ONE B200.  Real NCCL refuses two ranks on one device, so the
test builds tests/nccl_shim/nccl_shim.cu (an in-process stand-in for the
NCCL entry points partition.cu binds: every rank a host thread with its own
stream, every collective a rendezvous that checks the ranks issue the same
schedule, data moved stream-ordered) and points DPMRF_NCCL_LIB at it.  The
grouped halo send/recv windows, the counter all-reduce, the in-place
all-gathers and the side-stream exchange then execute for 2..8 ranks and
must reproduce the one-device optimize bit for bit (labels, mu, sigma, EM
trace), twice in a row per group."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


@pytest.fixture(scope="module")
def shim(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("shim") / "libnccl_shim.so")
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17",
                    "-Xcompiler", "-fPIC", "-shared", "-o", out,
                    os.path.join(HERE, "nccl_shim", "nccl_shim.cu")], check=True, timeout=300)
    return out


@pytest.mark.parametrize("size,block,brick,M,world,fixed,split", [
    (1024, 8, 0, 2, 2, 0, 1),
    (1024, 8, 0, 2, 3, 1, 1),
    (1024, 8, 0, 2, 4, 0, 0),
    (768, 8, 1, 5, 3, 0, 1),
    (2560, 8, 0, 2, 8, 1, 1),
    (2560, 8, 0, 2, 2, 0, 0),
])
def test_nccl_schedule_multi_rank(shim, size, block, brick, M, world, fixed, split):
    env = dict(os.environ, DPMRF_NCCL_LIB=shim, PYTHONPATH=ROOT)
    env["DPMRF_GROUP_SPLIT"] = str(split)  # 1: exchange overlapped with the interior hoods
    r = subprocess.run([sys.executable, os.path.join(HERE, "nccl_shim", "run_ranks.py"),
                        str(size), str(block), str(brick), str(M), str(world), str(fixed), "7"],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    rec = json.loads(r.stdout.strip().splitlines()[-1])
    assert rec["ok"] and rec["world"] == world
