"""Repeats bench.py's timed region (K asynchronous 32-spp C5 slabs after W warm-up
slabs, L2 flush between steps) R times in one process and prints each repetition's
device time: separates run-to-run variance of the asynchronous pipeline from box
variance.  python tools/timed_reps.py [reps] [steps]"""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
import torch
import paper_2011_03082_b200 as sb

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
r = sb.Renderer(0, "f32")
r.load_models_dir(bench.MODELS)
r.upload_scene(bench.build_scene_ours(sb))
be = bench._CudaBackend(0, r.stream)
with be.stream_ctx():
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
class A: pass
a = A(); a.warmup = int(os.environ.get("REPS_WARMUP", "3")); a.steps = steps
out = []
for k in range(reps):
    ms, stats, _ = bench.timed_slabs(r, be, None, 1, 0, a, 3 * 1920 * 1080, 32, 5000, flush)
    out.append(round(stats.segments / ms / 1e6, 4))
    print(f"rep {k}: {ms:.1f} ms, {stats.segments / ms / 1e6:.4f} Gseg/s", flush=True)
print(json.dumps({"gseg_s": out}))
