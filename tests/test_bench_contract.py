"""bench.py's reference arm runs on the host alone (the oracle timed on the box's
cores): its one JSON line must carry the keys the driver reads."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "0",
                          "--cpu-sample", "60000"], capture_output=True, text=True, timeout=600, check=True).stdout
    line = json.loads(out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] == "lifted SASS instructions/sec" and line["unit"] == "inst/s"
    assert line["value"] > 0 and line["higher_is_better"] is True and line["vs_baseline"] is None
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["cpu_baseline"]["value"] == line["value"] == line["e2e"]["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in line["config"]


def test_reference_arm_other_ranks_do_nothing():
    """under torchrun only rank 0 runs the CPU arm; the others exit 0 without output"""
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2"],
                         capture_output=True, text=True, timeout=120, check=True,
                         env={**__import__("os").environ, "RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}).stdout
    assert out.strip() == ""


def test_two_rank_bench_line_on_the_cpu_build(tmp_path):
    """`torchrun --nproc-per-node 2 bench.py --gpus 2` end to end without a GPU (CL_BENCH_SIM=1: one-lane CPU build of
    the device code, gloo): rank environment, LPT shard plan, the allgather of the match counters after every step,
    max-over-ranks timing and ONE JSON line from rank 0 with the contract's keys.  The whole-job counters must equal
    the single-rank run of the same corpus: the shards partition it."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ, CL_BENCH_SIM="1", MASTER_ADDR="127.0.0.1")
    common = ["bench.py", "--steps", "1", "--warmup", "1", "--insts", "60000", "--seed", "7"]
    lines = {}
    for n in (1, 2):
        cmd = ([sys.executable] if n == 1 else
               [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                "--master-port", "29641"]) + common + ["--gpus", str(n)]
        out = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        js = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
        assert len(js) == 1, out.stdout                      # rank 0 alone prints
        lines[n] = json.loads(js[0])
    two, one = lines[2], lines[1]
    assert two["n_gpus"] == 2 and two["scaling"] == "strong" and "dry run" in two["data"]
    for key in ("metric", "value", "unit", "steps", "warmup", "ms_per_step", "higher_is_better", "vs_baseline", "dtype", "config", "roofline", "gpu_launches"):
        assert key in two, key
    assert two["config"]["kernels"] == one["config"]["kernels"]
    assert two["config"]["sass_rank0"] < one["config"]["sass_rank0"]          # rank 0 holds its shard only
    for key in ("selected", "rewrites", "refused"):                            # counters are whole-job sums
        assert two["match_counts"][key] == one["match_counts"][key], key
    assert sum(two["match_counts"]["per_rank_selected"]) == one["match_counts"]["selected"]
