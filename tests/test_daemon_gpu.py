"""Context daemon analog: two processes
on one GPU.  The daemon owns the context slabs and executes the plan it
receives as JSON over a Unix socket; this process (the serving side) maps
the daemon's slab with CUDA IPC and, per pipeline stage, queues a device
wait on that stage's ready flag followed by a byte check of the stage's new
context -- which must be complete whenever its flag is up."""

import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import pytest

from paper_2311_15566_b200 import daemon, reshard

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]
ROOT = Path(__file__).resolve().parents[1]
SMALL = ("toy-bf16", 8, 8 * 1024 * 64, 1024)


@pytest.fixture()
def daemon_proc():
    path = os.path.join(tempfile.mkdtemp(), "ctx.sock")
    proc = subprocess.Popen([sys.executable, "-m", "paper_2311_15566_b200.daemon", "--socket", path],
                            cwd=ROOT, stdout=subprocess.PIPE, stderr=subprocess.PIPE)
    for _ in range(600):
        if os.path.exists(path) or proc.poll() is not None:
            break
        time.sleep(0.1)
    assert proc.poll() is None and os.path.exists(path), proc.stderr.read().decode()[-2000:]
    yield path
    if proc.poll() is None:
        proc.kill()
    proc.wait(timeout=30)


@pytest.mark.parametrize("old,new,u_max", [((1, 4, 2), (1, 2, 4), None), ((1, 2, 2), (1, 1, 4), 2.0e5),
                                           ((1, 2, 4), (2, 1, 4), 4e9)])
def test_daemon_migrates_and_consumer_waits_per_stage(daemon_proc, old, new, u_max):
    plan, layout, need, model, refs, mapping = reshard.make_reshard_problem(
        SMALL, old, new, 3, 64, u_max=u_max, with_mapping=True)
    req = daemon.migrate_request(plan, layout, need, model, mapping.assignment)
    client = daemon.DaemonClient(daemon_proc)
    try:
        done = client.migrate(req)
        client.release()
    finally:
        client.shutdown()
    assert done["op"] == "done" and done["error"] == 0 and done["progress"] == done["rounds"]
    assert done["mismatched_words"] == 0
    assert done["client_wait_timeouts"] == 0
    stages = {str(a.stage) for a in plan.actions if a.kind == "start_stage"}
    assert set(done["client_stage_mismatched_words"]) == stages
    assert all(v == 0 for v in done["client_stage_mismatched_words"].values())
