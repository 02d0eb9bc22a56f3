"""Per-call host timeline of bench.py's timed region (asynchronous C5 slabs): each
render call returns once its path supply is exhausted, so a stall shows up as one long
call. Prints per repetition the device time and the host duration of every call.
  python tools/first_rep_probe.py [reps] [steps]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
import paper_2011_03082_b200 as sb

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
r = sb.Renderer(0, "f32")
r.load_models_dir(bench.MODELS)
r.upload_scene(bench.build_scene_ours(sb))
be = bench._CudaBackend(0, r.stream)
n = 3 * 1920 * 1080
with be.stream_ctx():
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for k in range(reps):
    fsum, fsq = be.zeros(n), be.zeros(n)
    for i in range(3):
        r.render_device(sb.ST, 5000, i * 32, (i + 1) * 32, 1, True, fsum.data_ptr(), fsq.data_ptr(), asynchronous=True)
    r.read_stats()
    be.sync()
    stop = be.timer()
    calls = []
    for i in range(steps):
        t0 = time.perf_counter()
        with be.stream_ctx():
            flush.zero_()
        s0 = (3 + i) * 32
        r.render_device(sb.ST, 5000, s0, s0 + 32, 1, True, fsum.data_ptr(), fsq.data_ptr(), asynchronous=True)
        calls.append(round(1e3 * (time.perf_counter() - t0), 1))
    t0 = time.perf_counter()
    st = r.read_stats()
    drain = round(1e3 * (time.perf_counter() - t0), 1)
    ms = stop()
    print(f"rep {k}: {ms:.1f} ms ({st.segments / ms / 1e6:.3f} Gseg/s) calls {calls} drain {drain}", flush=True)
