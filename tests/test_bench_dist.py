"""bench.py's multi-rank code path on the CPU box: `--gpus N` re-launches itself under
torch.distributed.run, the ranks rendezvous over gloo, run the timed slabs and the
canonical-group frame through the stub slab renderer, reduce the films in fixed order
and rank 0 prints one JSON line (value null: nothing is measured without a GPU).
The frame film hash must not depend on the number of ranks."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(n):
    env = dict(os.environ, SST_BENCH_STUB="1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--steps", "3",
                          "--warmup", "3"], capture_output=True, text=True, env=env, timeout=600, check=True)
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout + out.stderr
    return json.loads(lines[0])


def test_bench_multi_rank_plumbing_gloo():
    one, two = _bench(1), _bench(2)
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["value"] is None and "unavailable" in two
    assert two["config"]["paths_per_step"] == 2 * one["config"]["paths_per_step"]
    # canonical sample groups + fixed-order reduce: bit-identical frame film for 1 and 2 ranks
    assert one["frame_stub"]["film_sha256"] == two["frame_stub"]["film_sha256"]
    assert one["frame_stub"]["paths"] == two["frame_stub"]["paths"]
