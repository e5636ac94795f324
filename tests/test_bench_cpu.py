"""bench.py host logic on CPU: the multi-GPU launcher, the reference arm's
chunking of the reference solve, and the torch.distributed plumbing (gloo,
world size 2)."""
import json
import os
import subprocess
import sys
import textwrap

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from cases import O  # noqa: E402


def test_gpus_n_without_enough_gpus_fails_loudly():
    # one process must never report an N-GPU number: with fewer visible GPUs
    # than --gpus the bench exits non-zero before measuring anything
    if bench.visible_gpus() >= 2:
        pytest.skip("host has >= 2 GPUs")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=300)
    assert p.returncode == 2
    assert "needs 2 visible GPUs" in p.stderr
    assert p.stdout.strip() == ""


def test_launcher_command_is_one_rank_per_gpu():
    cmd = bench.launcher_cmd(4, ["--gpus", "4", "--steps", "3"])
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--nnodes=1" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"]
    assert cmd[-5].endswith("bench.py")
    # a bare --n would be taken by torch.distributed.run itself
    assert bench.launcher_cmd(2, ["--n", "7", "--n=6"])[-3:] == ["--grid-n", "7", "--grid-n=6"]


@pytest.mark.parametrize("n,k", [(4, 1), (6, 5), (9, 20), (9, 200)])
def test_chunk_plan_covers_one_cycle_in_order(n, k):
    sched = O.build_schedule(n, 2)
    chunks, w, U = bench.chunk_plan(sched, k)
    assert len(chunks) == min(k, len(sched))
    assert [i for c in chunks for i in c] == list(range(len(sched)))
    assert all(c for c in chunks)
    assert U == bench.units(n) == O.closed_form_work_units(n, 2)


def test_dist_plumbing_gloo_two_ranks(tmp_path):
    script = tmp_path / "d.py"
    script.write_text(textwrap.dedent(f"""
        import sys, json
        sys.path.insert(0, {ROOT!r})
        import bench
        world, rank, local = bench.dist_env()
        d = bench.Dist(world, rank, local)
        d.barrier()
        mx = d.reduce(float(rank + 1), "max")
        sm = d.reduce(float(rank + 1), "sum")
        if rank == 0:
            print(json.dumps({{"world": world, "max": mx, "sum": sm}}))
        d.close()
    """))
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", f"--master-port={bench.free_port()}", str(script)],
                       capture_output=True, text=True, timeout=300, env=env)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads([x for x in p.stdout.splitlines() if x.startswith("{")][-1])
    assert line == {"world": 2, "max": 2.0, "sum": 3.0}


@pytest.mark.skipif(O.ref_lib() is None, reason="reference build unavailable")
def test_reference_arm_runs_one_full_cycle_of_the_same_problem():
    env = dict(os.environ, OMP_NUM_THREADS="2")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--n", "5",
                        "--steps", "4", "--warmup", "3"], capture_output=True, text=True, timeout=300, env=env)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["steps"] == 4 and line["value"] > 0
    assert line["config"]["n"] == 5 and line["cpu_baseline"]["cores"] == 2
    assert line["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.skipif(O.ref_lib() is None, reason="reference build unavailable")
def test_reference_arm_under_torchrun_prints_one_line_from_rank_0():
    # the driver launches the reference arm like our own (torchrun, N ranks):
    # rank 0 alone runs and prints; no GPU per rank, no process group needed
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    env.pop("OMP_NUM_THREADS", None)  # (torch.distributed.run then sets 1 per process)
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", f"--master-port={bench.free_port()}",
                        os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--grid-n", "4",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=300, env=env)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [x for x in p.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["value"] > 0
    # torch.distributed.run sets OMP_NUM_THREADS=1 per process; rank 0 takes
    # the host's cores back
    assert line["cpu_baseline"]["cores"] == bench.host_cores()


@pytest.mark.skipif(O.ref_lib() is None, reason="reference build unavailable")
def test_ref_session_cycle_equals_reference_single_cycle():
    # the steppable session runs exactly the reference's cycle: its state after
    # all schedule steps + the recurrence matches solve()'s first cycle
    n = 4
    g = O.make_grid(3, n)
    f = O.fill("poisson3d", g)
    sess = O.RefSession(g, O.all_dirichlet(0.0), f)
    sess.begin_cycle(False)
    for i in range(len(sess.schedule)):
        assert sess.step(i) == 0
    rmax = sess.recurrence()
    ref = O.solve(g, O.all_dirichlet(0.0), f, tol=1e-10, max_cycles=1, impl="ref")
    assert rmax / float(abs(f).max()) == ref.rows[0][2]
