#!/usr/bin/env python
"""Benchmark of the north-star path: CVAE sphere tracing (SDF safe radius -> CVAE
sphere step -> NEE -> continue/exit) on the config-5 teaser scene of BASELINE.json
(1920x1080, four media sigma_t = 20/40/80/160, g = 0.8), one JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--spp-per-step S] [--impl ours|reference]

--gpus N > 1 without a torchrun environment re-launches this script under
`python -m torch.distributed.run --nproc-per-node N` (one rank per GPU, NCCL).

A step = one sample slab of S spp over every pixel and channel of the 1080p frame
(3 * 1920 * 1080 * S light paths) on each rank; ranks render disjoint sample slabs
(weak scaling) and their films (FP64 sum and sum of squares) are reduced to rank 0 in
FIXED rank order (paper_2011_03082_b200/dist.py ordered_film_sum) at the end of the
timed region. value = light-path segments (sphere steps + delta-tracking events,
counted on the device) of all ranks / max-over-ranks time.

frame_time_s: one complete 1080p @ 5000 spp frame on all N GPUs (canonical sample
groups, fixed-order reduce), timed on the device, max over ranks; frame_film_sha256 is
the hash of the reduced film -- identical for every N by construction.

--impl reference runs the reference's own CPU implementation (oracle/_ref: the
reference sources + the reference-composed integrator) on the host cores, rank 0 only.

Without a CUDA device (the CPU dev box; or with SST_BENCH_STUB=1) the multi-rank plumbing (launch, gloo
rendezvous, ordered film reduce, max-over-ranks timing) runs with a stub slab renderer
and the line reports value null with "unavailable": nothing is measured.
"""
from __future__ import annotations

import argparse
import ctypes as C
import hashlib
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
MODELS = os.path.join(ROOT, "tests", "golden", "models")
PROFILES = os.path.join(ROOT, "profiles")

FRAME_SPP = 5000
W_FRAME, H_FRAME = 1920, 1080
METRIC = "light-path segments/sec"
WORKLOAD = ("c5 teaser (BASELINE.json configs[4]): 4 unit icospheres(3), sigma_t 20/40/80/160, "
            "g=0.8, phi=(0.99999,0.99995,0.975), point light, 1920x1080, ST+NEE")
DATA = ("synthetic: procedural icosphere meshes, GPU-built conservative SDFs (res 64), "
        "deterministic desk-scale CVAE weights trained by the reference's train_model")


def mlp_flops(dl, dp, de):
    """Algorithmic FLOPs of the decoders: 2 x MACs x decodes."""
    return 2.0 * (112 * dl + 480 * dp + 640 * de)


# Algorithmic per-unit work of each wavefront kernel (counted from the
# device counters of the measured slab):
#   wf_logic  HBM (layout basis): per slot visit the path state it must read (x,L 16 +
#             w,r 16 + rng 8 + meta 16 = 56 B; meta.z holds the trace-queue position while
#             a traversal is queued), write back and its live-list entry (60 B in all);
#             per flight it sends to the trace kernel the 36 B ray record + the 12 B
#             result it reads back next pass; per fresh path the
#             camera-ray result and direction (28 B); per delta-tracking event its NEE
#             record + queue entry (36 B); per sphere request a queue entry (4 B).
#   wf_logic  HBM (SURVEY §8(d) basis, `frac_survey`): 96 B per segment (48 B state read
#             + 48 B written).
#   wf_trace  FP32: per interior node 2 slab tests = 12 FFMA + 12 min/max = 36 FLOP;
#             per Moller-Trumbore test 51 FLOP (2 cross, 4 dot, rcp, 3 mul, 3 sub).
#   wf_shadow FP32: 51 FLOP per light-grid triangle test.
#   wf_sphere FP32: decoder MLP FLOPs 2*(112 nL + 480 nP + 640 nE).
NODE_FLOP, TRI_FLOP = 36.0, 51.0
LOGIC_BYTES_PER_SLOT, LOGIC_BYTES_PER_FLIGHT, LOGIC_BYTES_PER_FRESH = 116.0, 48.0, 28.0
NEE_RECORD_BYTES, SPHERE_QUEUE_BYTES = 36.0, 4.0
SURVEY_BYTES_PER_SEGMENT = 96.0


def logic_bytes(k):
    """Algorithmic HBM bytes of the logic kernel over a measured slab (device counters)."""
    flights = max(0.0, float(k.traversals) - float(k.paths) / 3.0)
    return (LOGIC_BYTES_PER_SLOT * k.wavefront_slot_visits + LOGIC_BYTES_PER_FLIGHT * flights
            + LOGIC_BYTES_PER_FRESH * k.paths + NEE_RECORD_BYTES * k.pt_events
            + SPHERE_QUEUE_BYTES * k.sphere_steps)


def source_hash() -> str:
    """Hash of the CUDA/C++ sources and public headers the library is built from; stamps
    ncu traffic files so a stale capture is never reported against a newer build."""
    h = hashlib.sha256()
    dirs = [os.path.join(ROOT, "paper_2011_03082_b200", "csrc"), os.path.join(ROOT, "include")]
    for d in dirs:
        for f in sorted(os.listdir(d)):
            if f.endswith((".cu", ".cuh", ".cpp", ".h", ".hpp")):
                h.update(f.encode())
                with open(os.path.join(d, f), "rb") as fh:
                    h.update(fh.read())
    return h.hexdigest()[:16]


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or platform.machine()


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during the timed region."""
    NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
             0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
             0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz, self.ok = [], set(), None, False
        if index is None:
            self.err = "no GPU"
            self._stop = threading.Event()
            return
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                bits = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for b, n in self.NAMES.items():
                    if bits & b and b != 0x1:
                        self.reasons.add(n)
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": "NVML unavailable"}
        s = self.samples or [0]
        return {"sm_mhz": float(np.median(s)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def nvml_index(local):
    cvd = os.environ.get("CUDA_VISIBLE_DEVICES")
    if cvd:
        parts = cvd.split(",")
        if local < len(parts) and parts[local].strip().isdigit():
            return int(parts[local])
    return local


def build_scene_ours(sb):
    mesh = sb.make_icosphere(3, 1.0)
    return sb.c5_scene(mesh, W_FRAME, H_FRAME)


def relaunch(n: int) -> int:
    """--gpus N outside torchrun: one rank per GPU under torch.distributed.run."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ------------------------------------------------------------------ CPU reference arm
def cpu_reference_rate(seconds: float, seed: int = 99, threads: int | None = None):
    """Times the reference CPU path (oracle/_ref) on a bounded random sample of the
    workload's light paths. Returns (run, n, threads); run(n) -> (dt, stats, keys, rad, seg, exit_state)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import reflib
    from paper_2011_03082_b200 import abi
    from paper_2011_03082_b200.scene import SdfGrid, c5_scene
    threads = threads or os.cpu_count() or 1
    os.environ["SST_THREADS"] = str(threads)
    P, T = reflib.make_mesh("icosphere", 3, 1.0)
    sdfs = []
    for i in range(4):  # the reference's own build_sdf on each placed object
        off = np.array([-3.3 + 2.2 * i, 0.0, 0.0])
        sdfs.append(SdfGrid(*reflib.build_sdf(P + off, T, 64)))
    sc = c5_scene((P, T), W_FRAME, H_FRAME)
    for i, o in enumerate(sc.objects):
        o.sdf = sdfs[i]
    desc = sc.to_desc()
    rs = reflib.Scene(C.byref(desc))
    models = reflib.Models(MODELS)
    rng = np.random.default_rng(seed)

    def run(n):
        pix = rng.integers(0, W_FRAME * H_FRAME, n).astype(np.uint32)
        smp = rng.integers(0, FRAME_SPP, n).astype(np.uint32)
        ch = rng.integers(0, 3, n).astype(np.uint8)
        st = abi.PathStats()
        t0 = time.perf_counter()
        rad, seg, ex = rs.trace_paths(models, 1, 1, 1, pix, smp, ch, st, exit_state=True)
        return time.perf_counter() - t0, st, (pix, smp, ch), rad, seg, ex

    run._keep = (desc, rs, models)
    dt = run(4000)[0]  # calibration
    rate_paths = 4000 / max(dt, 1e-6)
    n = int(max(4000, rate_paths * seconds))
    return run, n, threads


def bench_reference(args, world, rank):
    if rank != 0:
        return
    run, n, threads = cpu_reference_rate(args.ref_seconds)
    for _ in range(args.warmup):
        run(max(1000, n // 10))
    tot_seg = 0
    tot_t = 0.0
    for _ in range(args.steps):
        dt, st = run(n)[:2]
        tot_seg += st.segments
        tot_t += dt
    value = tot_seg / tot_t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "segments/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": DATA, "config": {"workload": WORKLOAD, "paths_per_step": n,
                                 "sample": f"{n} uniformly random (pixel, sample, channel) paths of the frame per step"},
        "cpu_baseline": {"value": value, "unit": "segments/s", "cores": threads, "kind": "reference",
                         "sample": f"{n} random light paths of the 1080p frame per step, {args.steps} steps",
                         "cpu": cpu_model()},
        "e2e": {"value": value, "unit": "segments/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def load_traffic():
    """ncu DRAM bytes per launch (profiles/traffic.json), only if it was captured from
    the sources this library is built from (src_hash stamp)."""
    p = os.path.join(PROFILES, "traffic.json")
    if not os.path.exists(p):
        return None, "profiles/traffic.json missing"
    try:
        t = json.load(open(p))
    except Exception as e:  # noqa: BLE001
        return None, f"unreadable: {e}"
    if t.get("src_hash") != source_hash():
        return None, f"stale: captured from sources {t.get('src_hash')}, built from {source_hash()}"
    return t, None


# ------------------------------------------------------------------ device backends
class _CudaBackend:
    """Device film tensors on the context's stream, CUDA-event timing."""

    def __init__(self, local, stream):
        import torch
        self.torch = torch
        self.dev = torch.device("cuda", local)
        self.stream = torch.cuda.ExternalStream(stream)

    def zeros(self, n):
        with self.torch.cuda.stream(self.stream):
            return self.torch.zeros(n, dtype=self.torch.float64, device=self.dev)

    def timer(self):
        torch = self.torch
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(self.stream)

        def stop():
            ev1.record(self.stream)
            torch.cuda.synchronize()
            return ev0.elapsed_time(ev1)

        return stop

    def sync(self):
        self.torch.cuda.synchronize()

    def stream_ctx(self):
        return self.torch.cuda.stream(self.stream)


class _HostBackend:
    """CPU tensors + wall clock (the gloo plumbing check without a GPU)."""

    def __init__(self):
        import torch
        self.torch = torch
        self.dev = torch.device("cpu")

    def zeros(self, n):
        return self.torch.zeros(n, dtype=self.torch.float64)

    def timer(self):
        t0 = time.perf_counter()
        return lambda: 1e3 * (time.perf_counter() - t0)

    def sync(self):
        pass

    def stream_ctx(self):
        import contextlib
        return contextlib.nullcontext()


class _PlumbingStub:
    """Stand-in slab renderer for hosts without a CUDA device: writes a deterministic
    per-(pixel, sample, channel) value pattern into the film so the ordered reduce is
    exercised on real numbers. Not a renderer; the bench reports no value with it."""

    def __init__(self, width, height):
        from paper_2011_03082_b200 import abi
        self.abi = abi
        self.n = width * height * 3
        self.pending = abi.PathStats()

    def render_device(self, integrator, spp_total, s0, s1, seed, nee, sum_ptr, sq_ptr, stats=None,
                      asynchronous=False):
        fs = np.ctypeslib.as_array((C.c_double * self.n).from_address(sum_ptr))
        fq = np.ctypeslib.as_array((C.c_double * self.n).from_address(sq_ptr))
        k = np.arange(self.n, dtype=np.uint64)
        with np.errstate(over="ignore"):
            for s in range(s0, s1):
                h = (k * np.uint64(0x9E3779B97F4A7C15) + np.uint64(s) * np.uint64(0xBF58476D1CE4E5B9)) >> np.uint64(40)
                v = h.astype(np.float64) / float(1 << 24)
                fs += v
                fq += v * v
        st = self.pending if asynchronous else (stats if stats is not None else self.abi.PathStats())
        st.paths += self.n * (s1 - s0)
        st.segments += 2 * self.n * (s1 - s0)
        return None if asynchronous else st

    def read_stats(self):
        st, self.pending = self.pending, self.abi.PathStats()
        return st


def _max_over_ranks(dist, be, vals):
    t = be.torch.tensor(vals, dtype=be.torch.float64, device=be.dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def _sum_over_ranks(dist, be, vals):
    t = be.torch.tensor([int(v) for v in vals], dtype=be.torch.int64, device=be.dev)
    if dist:
        dist.all_reduce(t)
    return t.tolist()


def _film_hash(fsum, fsq):
    h = hashlib.sha256()
    h.update(fsum.cpu().numpy().tobytes())
    h.update(fsq.cpu().numpy().tobytes())
    return h.hexdigest()[:16]


def timed_slabs(r, be, dist, world, rank, args, n_values, S, spp_total, flush=None):
    """W warm-up + K timed sample slabs (asynchronous enqueue), then the fixed-order film
    reduce inside the timed region. Returns (ms max over ranks, stats, film hash)."""
    from paper_2011_03082_b200 import ST
    from paper_2011_03082_b200.dist import ordered_film_sum
    fsum, fsq = be.zeros(n_values), be.zeros(n_values)

    def one(step):
        if flush is not None:
            with be.stream_ctx():
                flush.zero_()  # evict L2 between steps (inputs are L2-resident by design)
        s0 = (step * world + rank) * S
        r.render_device(ST, spp_total, s0, s0 + S, 1, True, fsum.data_ptr(), fsq.data_ptr(), asynchronous=True)

    for i in range(args.warmup):
        one(i)
    r.read_stats()
    with be.stream_ctx():
        # one untimed reduce first: its output buffers come from the caching allocator
        # afterwards (a first-time cudaMalloc inside the timed region cost up to ~10% of a
        # 10-slab measurement)
        ordered_film_sum({rank: (fsum, fsq)}, list(range(world)))
        fsum.zero_()
        fsq.zero_()
    if dist:
        dist.barrier()
    be.sync()
    stop = be.timer()
    for i in range(args.steps):
        one(args.warmup + i)
    stats = r.read_stats()  # joins the pipeline and synchronises the context
    with be.stream_ctx():
        red = ordered_film_sum({rank: (fsum, fsq)}, list(range(world)))
    ms = stop()
    if dist:
        dist.barrier()
    (ms,) = _max_over_ranks(dist, be, [ms])
    fh = _film_hash(*red) if red is not None else None
    return ms, stats, fh


def timed_frame(r, be, dist, world, rank, n_values, spp):
    """One complete frame of `spp` samples on all ranks: canonical sample groups
    (dist.FRAME_GROUPS), each into its own film, fixed-order reduce to rank 0."""
    from paper_2011_03082_b200 import ST
    from paper_2011_03082_b200.dist import group_owners, group_slab, groups_of_rank, ordered_film_sum
    mine = list(groups_of_rank(rank, world))
    films = {g: (be.zeros(n_values), be.zeros(n_values)) for g in mine}
    with be.stream_ctx():  # untimed reduce first: its buffers come from the allocator cache
        ordered_film_sum(films, group_owners(world))
    if dist:
        dist.barrier()
    be.sync()
    stop = be.timer()
    for g in mine:
        s0, s1 = group_slab(g, spp)
        fs, fq = films[g]
        r.render_device(ST, spp, s0, s1, 1, True, fs.data_ptr(), fq.data_ptr(), asynchronous=True)
    stats = r.read_stats()
    with be.stream_ctx():
        red = ordered_film_sum(films, group_owners(world))
    ms = stop()
    if dist:
        dist.barrier()
    (ms,) = _max_over_ranks(dist, be, [ms])
    seg, paths = _sum_over_ranks(dist, be, [stats.segments, stats.paths])
    out = {"frame": f"{W_FRAME}x{H_FRAME} @ {spp} spp" if n_values == 3 * W_FRAME * H_FRAME else None,
           "frame_time_s": ms / 1e3, "segments": seg, "paths": paths,
           "groups": len(group_owners(world)), "reduce": "fixed group order (dist.ordered_film_sum)"}
    if red is not None:
        out["film_sha256"] = _film_hash(*red)
    del films
    return out


def bench_stub(args, world, rank):
    """No CUDA device: run the multi-rank plumbing (gloo) with the stub slab renderer."""
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    be = _HostBackend()
    w, h = 64, 36
    r = _PlumbingStub(w, h)
    S = args.spp_per_step
    spp_total = max(FRAME_SPP, (args.warmup + args.steps) * world * S)
    ms, stats, fh = timed_slabs(r, be, dist, world, rank, args, 3 * w * h, S, spp_total)
    frame = timed_frame(r, be, dist, world, rank, 3 * w * h, 64)
    seg_all, paths_all = _sum_over_ranks(dist, be, [stats.segments, stats.paths])
    if rank == 0:
        line = {"metric": METRIC, "value": None, "unit": "segments/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "none (plumbing stub)",
                "unavailable": "no CUDA device on this host: the multi-rank plumbing (launch, gloo rendezvous, "
                               "fixed-order film reduce, max-over-ranks timing) ran with a stub slab renderer; "
                               "nothing was measured",
                "config": {"workload": WORKLOAD, "stub_frame": f"{w}x{h}", "spp_per_step_per_gpu": S,
                           "paths_per_step": int(paths_all / args.steps), "segments": int(seg_all),
                           "parallelism": f"sample slabs per rank x{world} + fixed-order film reduce"},
                "film_sha256": fh, "frame_stub": frame, "gpu_launches": 0}
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def bench_ours(args, world, rank, local):
    import torch
    if not torch.cuda.is_available() or os.environ.get("SST_BENCH_STUB") == "1":
        return bench_stub(args, world, rank)

    import paper_2011_03082_b200 as sb
    from paper_2011_03082_b200 import abi

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    r = sb.Renderer(local, "f32")
    r.load_models_dir(MODELS)
    scene = build_scene_ours(sb)
    r.upload_scene(scene)
    info = r.scene_info()
    be = _CudaBackend(local, r.stream)
    n_pix = W_FRAME * H_FRAME
    S = args.spp_per_step
    total_steps = args.warmup + args.steps
    # sample indices past the 5000-spp frame are further samples of the same pixels
    # (keyed RNG): the per-path work distribution is the frame's
    spp_total = max(FRAME_SPP, (total_steps + 1) * world * S)
    # FFMA roofline denominator (measured once, before the timed region)
    peak_lib = C.CDLL(os.path.join(ROOT, "paper_2011_03082_b200", "libsst_peak.so"))
    peak_lib.sst_peak_ffma_tflops.restype = C.c_double
    peak_lib.sst_peak_ffma_tflops.argtypes = [C.c_int, C.c_int]
    fp32_peak = peak_lib.sst_peak_ffma_tflops(local, 5)
    props = torch.cuda.get_device_properties(local)
    with be.stream_ctx():
        flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > L2

    with ClockSampler(nvml_index(local)) as clocks:
        ms, stats, film_hash = timed_slabs(r, be, dist, world, rank, args, 3 * n_pix, S, spp_total, flush)
    seg_all, paths_all, sphere_all, events_all, dl, dp, de = _sum_over_ranks(
        dist, be, [stats.segments, stats.paths, stats.sphere_steps, stats.pt_events, stats.decodes_length,
                   stats.decodes_path, stats.decodes_event])
    value = seg_all / (ms / 1e3)
    ms_step = ms / args.steps
    flops_all = mlp_flops(dl, dp, de)
    # SURVEY §8(d) FP32 FFMA peak: SMs x 128 lanes x 2 x max SM clock
    survey_fp32_peak = props.multi_processor_count * 128 * 2 * (clocks.max_mhz or 1965) * 1e6 / 1e12

    # ---- per-kernel roofline: one more slab with every launch bracketed by CUDA events
    # on its own stream (synchronous per iteration, so outside the timed region)
    hbm_peak = 6551.7
    try:
        hbm_peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:  # noqa: BLE001
        pass
    r.kernel_timing(True)
    kst = abi.PathStats()
    s0k = total_steps * world * S + rank * S
    ksum, ksq = be.zeros(3 * n_pix), be.zeros(3 * n_pix)
    r.render_device(sb.ST, spp_total, s0k, s0k + S, 1, True, ksum.data_ptr(), ksq.data_ptr(), stats=kst)
    kt = r.kernel_timing(False)
    del ksum, ksq
    tri_trace = kst.triangle_tests - kst.shadow_triangle_tests
    kdef = {
        "wf_logic": ("hbm", logic_bytes(kst) / 1e9, hbm_peak, "GB/s"),
        "wf_trace": ("fp32", (NODE_FLOP * kst.node_visits + TRI_FLOP * tri_trace) / 1e12, fp32_peak, "TFLOP/s"),
        "wf_shadow": ("fp32", TRI_FLOP * kst.shadow_triangle_tests / 1e12, fp32_peak, "TFLOP/s"),
        "wf_sphere": ("fp32", mlp_flops(kst.decodes_length, kst.decodes_path, kst.decodes_event) / 1e12,
                      fp32_peak, "TFLOP/s"),
    }
    tot_ms = sum(v[0] for v in kt.values())
    kernels = {}
    for k, (ms_k, n_k) in kt.items():
        if n_k == 0:
            continue
        e = {"ms": ms_k, "launches": n_k, "avg_us": 1e3 * ms_k / n_k, "share": ms_k / tot_ms if tot_ms else None}
        if k in kdef and ms_k > 0:
            bound, work, peak, unit = kdef[k]
            ach = work / (ms_k / 1e3)
            e.update({"bound": bound, "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak})
        kernels[k] = e
    dominant = max((k for k in kernels if k in kdef), key=lambda k: kernels[k]["ms"], default=None)
    traffic, traffic_note = load_traffic()
    dom_traffic = None
    if traffic and dominant:
        dom_traffic = traffic.get("kernels", {}).get(dominant, {}).get("dram_bytes_per_launch")
    frac_survey = None
    if "wf_logic" in kernels:
        lg = kernels["wf_logic"]
        ach_s = SURVEY_BYTES_PER_SEGMENT * kst.segments / (lg["ms"] / 1e3) / 1e9
        sp = kernels.get("wf_sphere")
        dec = mlp_flops(kst.decodes_length, kst.decodes_path, kst.decodes_event) / 1e12
        frac_survey = {
            "wf_logic": {"achieved": ach_s, "unit": "GB/s", "peak": hbm_peak, "frac": ach_s / hbm_peak,
                         "def": "96 B per segment (SURVEY §8(d): 48 B state read + 48 B written) x segments of "
                                "the slab / summed wf_logic launch time"},
            "wf_sphere_decoder": ({"achieved": dec / (sp["ms"] / 1e3), "unit": "TFLOP/s", "peak": survey_fp32_peak,
                                   "frac": dec / (sp["ms"] / 1e3) / survey_fp32_peak,
                                   "def": "decoder MLP FLOPs / summed wf_sphere launch time vs SMs x 128 x 2 x "
                                          "sm_max_mhz (SURVEY §8(d))"} if sp else None),
            "decoder_whole_render": {"achieved": flops_all / (ms / 1e3) / 1e12 / world, "unit": "TFLOP/s",
                                     "peak": survey_fp32_peak,
                                     "frac": flops_all / (ms / 1e3) / 1e12 / world / survey_fp32_peak,
                                     "def": "decoder MLP FLOPs of the timed region per GPU / timed-region "
                                            "time (SURVEY §8(d))"},
        }

    # ---- one complete 1080p @ 5000 spp frame on all ranks (measured, not extrapolated)
    frame = None
    if not args.no_frame:
        with ClockSampler(nvml_index(local)) as fclk:
            frame = timed_frame(r, be, dist, world, rank, 3 * n_pix, FRAME_SPP)
        frame["clocks"] = fclk.summary()
        frame["segments_per_s"] = frame["segments"] / frame["frame_time_s"]

    # ---- e2e: the public host-buffer API per step (scene upload + render + film D2H)
    e2e = None
    if not args.no_e2e:
        film = sb.Film(W_FRAME, H_FRAME, np.zeros(3 * n_pix), np.zeros(3 * n_pix), 0)
        est = abi.PathStats()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for i in range(args.steps):
            r.upload_scene(scene)
            s0 = ((args.warmup + i) * world + rank) * S
            r.render_film(sb.ST, spp_total, 1, True, s0, s0 + S, film, est)
        t_e2e = time.perf_counter() - t0
        (t_e2e,) = _max_over_ranks(dist, be, [t_e2e])
        (e_seg,) = _sum_over_ranks(dist, be, [est.segments])
        e2e = {"value": e_seg / t_e2e, "unit": "segments/s",
               "h2d_bytes_per_step": int(info["h2d_bytes"]),
               "d2h_bytes_per_step": int(2 * 3 * n_pix * 8),
               "path": "sst_gpu_upload_scene + sst_gpu_render(SST_PTR_HOST) per step, per rank"}

    # ---- CPU reference baseline + per-path parity on the same keys (rank 0, N = 1)
    cpu = parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        run, n, threads = cpu_reference_rate(args.ref_seconds / 2)
        dt, st, keys, o_rad, o_seg, o_ex = run(n)
        cpu = {"value": st.segments / dt, "unit": "segments/s", "cores": threads, "kind": "reference",
               "cpu": cpu_model(),
               "sample": f"{n} uniformly random (pixel, sample, channel) light paths of the 1080p frame "
                         f"({st.segments} segments, {dt:.1f} s), reference sources + reference-composed integrator"}
        def agree(g_rad, g_seg, o_rad, o_seg, g_ex, o_ex):
            same = g_seg == o_seg
            out = {"paths": int(len(o_seg)), "segments_equal": float(same.mean())}
            for rt in (1e-5, 1e-4, 1e-3):
                ok = same & (np.abs(g_rad - o_rad) <= 1e-12 + rt * np.abs(o_rad))
                out[f"agree_rtol_{rt:g}"] = float(ok.mean())
            # per-path exit state: max(|dx| / max(|x|, 1), |dw|) of the final position / direction
            dx = np.linalg.norm(g_ex[:, :3] - o_ex[:, :3], axis=1) / np.maximum(
                np.linalg.norm(o_ex[:, :3], axis=1), 1.0)
            e = np.maximum(dx, np.linalg.norm(g_ex[:, 3:] - o_ex[:, 3:], axis=1))
            for rt in (1e-6, 1e-5, 1e-4):
                out[f"exit_state_rtol_{rt:g}"] = float((e <= rt).mean())
            return out

        gst = abi.PathStats()
        g_rad, g_seg, g_ex = r.trace_paths(sb.ST, 1, 1, *keys, stats=gst, exit_state=True)
        fp32 = agree(g_rad, g_seg, o_rad, o_seg, g_ex, o_ex)
        fp32.update({"engine": "wavefront FP32 (sst_gpu_trace_paths: the bench's kernels)",
                     "segments_total_gpu": int(gst.segments), "segments_total_ref": int(st.segments)})
        # the FP64 parity build of the same kernels on the first 400k of the same keys
        m = min(n, 400_000)
        r.set_precision("f64")
        try:
            d_rad, d_seg, d_ex = r.trace_paths(sb.ST, 1, 1, *(k[:m] for k in keys), exit_state=True)
        finally:
            r.set_precision("f32")
        fp64 = agree(d_rad, d_seg, o_rad[:m], o_seg[:m], d_ex, o_ex[:m])
        fp64["engine"] = "wavefront FP64 parity build (-fmad=false)"
        parity = {"reference": "oracle/_ref (reference sources + reference-composed integrator), same keys as "
                               "cpu_baseline", "fp32": fp32, "fp64_parity_mode": fp64,
                  "agreement": fp32["exit_state_rtol_0.0001"],
                  "agreement_def": "FP32 production path: fraction of paths whose exit state (final position "
                                   "and direction) matches the reference within 1e-4 relative -- the north "
                                   "star's bar; radiance rates beside it (DESIGN.md §4: FP32 state drift x "
                                   "sigma_t bounds the radiance 1e-4 rate; the FP64 parity build meets 1e-5 on "
                                   "every path)"}

    # ---- secondary configs (rank 0, N = 1; not the headline metric)
    extra = None
    if rank == 0 and world == 1 and not args.no_extra:
        extra = run_extras(r, sb, abi, scene, local, args)
        r.upload_scene(scene)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "segments/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": DATA,
            "sphere_steps_per_s": sphere_all / (ms / 1e3),
            "pt_events_per_s": events_all / (ms / 1e3),
            "paths_per_s": paths_all / (ms / 1e3),
            "frame_time_s": frame["frame_time_s"] if frame else None,
            "frame_film_sha256": frame.get("film_sha256") if frame else None,
            "config": {
                "workload": WORKLOAD, "spp_per_step_per_gpu": S, "paths_per_step": int(paths_all / args.steps),
                "frame_spp": FRAME_SPP,
                "sphere_steps": int(sphere_all), "pt_events": int(events_all),
                "l2": "flushed between steps by a 256 MB device write (scene is L2-resident by design)",
                "parallelism": f"sample slabs per rank x{world}" + (" + fixed-order film reduce (NCCL p2p)"
                                                                    if world > 1 else ""),
                "bvh_nodes": info["bvh_nodes"], "triangles": info["triangles"],
                "timed_film_sha256": film_hash,
            },
            "frame": frame,
            "roofline": {
                "bound": kernels[dominant]["bound"] if dominant else None,
                "achieved": kernels[dominant]["achieved"] if dominant else None,
                "peak": kernels[dominant]["peak"] if dominant else None,
                "unit": kernels[dominant]["unit"] if dominant else None,
                "frac": kernels[dominant]["frac"] if dominant else None,
                "traffic": dom_traffic,
                "traffic_note": traffic_note or f"profiles/traffic.json src_hash {source_hash()} (matches this build)",
                "frac_survey": frac_survey,
                "kernel": f"k_{dominant} (wavefront)" if dominant else None,
                "share_of_kernel_time": kernels[dominant]["share"] if dominant else None,
                "achieved_def": "algorithmic work of the measured slab (device counters; bench.py NODE_FLOP/TRI_FLOP/"
                                "LOGIC_BYTES_PER_SLOT) / summed CUDA-event duration of that kernel's launches on "
                                "their stream (one extra slab after the timed region)",
                "peak_source": f"HBM: MEASURED_PEAKS.json hbm_gbs; FP32: measured FFMA throughput (csrc/peak.cu) "
                               f"{fp32_peak:.1f} TFLOP/s on this GPU (MEASURED_PEAKS.json has no FP32 figure); "
                               f"frac_survey uses SURVEY §8(d)'s {survey_fp32_peak:.1f} TFLOP/s",
                "kernels": kernels,
                "src_hash": source_hash(),
            },
            "parity": parity,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": sum(n for _, n in kt.values()) * args.steps,
            "gpu_launches_def": "kernel launches of one slab (counted by the library's per-kernel timing pass) x steps",
            "extra": extra,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()  # rank 0 may still be on the extras / JSON line
    r.close()
    if dist:
        dist.destroy_process_group()


def run_extras(r, sb, abi, scene, local, args):
    """Secondary BASELINE.json configs at their stated sizes, each with its own clocks."""
    import torch
    extra = {}
    mesh = sb.make_icosphere(3, 1.0)
    for name, integ in (("c1_st_nee", sb.ST), ("c2_pt_nee", sb.PT)):
        r.upload_scene(sb.c1_scene(mesh, 256, 256))
        r.render_film(integ, 64, 1, True, 0, 8)  # warm-up
        est = abi.PathStats()
        with ClockSampler(nvml_index(local)) as ck:
            r.render_film(integ, 64, 1, True, 0, 64, stats=est)
        extra[name] = {"frame": "256x256 @ 64 spp (full config)", "frame_ms": est.device_ms,
                       "segments_per_s": est.segments / (est.device_ms / 1e3),
                       "segments_per_path": est.segments / est.paths, "clocks": ck.summary()}
    # config 4: the full 1e8-walk training-data job, records into device memory
    n4 = 100_000_000 if not args.quick_extra else 8_000_000
    out = torch.empty(n4 * 52, dtype=torch.uint8, device="cuda")
    L = abi.lib()
    r.generate_dataset(200000, seed=7)  # warm-up
    dst = abi.DatasetStats()
    with ClockSampler(nvml_index(local)) as ck:
        abi.check(L.sst_gpu_generate_dataset(r.h, n4, 0.0, 200.0, -1.0, 1.0, 0, -5.0, -0.5, 7, 0,
                                             C.c_void_p(out.data_ptr()), abi.SST_PTR_DEVICE, C.byref(dst)))
    extra["c4_dataset"] = {"walks": int(dst.walks), "time_s": dst.device_ms / 1e3,
                           "walks_per_s": dst.walks / (dst.device_ms / 1e3),
                           "events_per_s": dst.events / (dst.device_ms / 1e3),
                           "sample": f"{n4:.0e} walks (the full config-4 job), sigma_t U[0,200], g U[-1,1], "
                                     "phi 1-10^U[-5,-0.5], records written to HBM",
                           "clocks": ck.summary()}
    del out
    # config 3: density-doubling sweep on the SDF-boundary bumpy-sphere scene, 512x512 @ 1000 spp
    bumpy = sb.make_bumpy_sphere(4, 1.0, 0.2, 3.0)
    spp3 = 1000 if not args.quick_extra else 8
    sweep = []
    for sig in (10.0, 20.0, 40.0, 80.0, 160.0):
        r.upload_scene(sb.c3_scene(bumpy, sig))
        row = {"sigma_t": sig}
        for iname, integ in (("st", sb.ST), ("pt", sb.PT)):
            r.render_film(integ, spp3, 1, True, 0, 1)  # warm-up
            est = abi.PathStats()
            with ClockSampler(nvml_index(local)) as ck:
                r.render_film(integ, spp3, 1, True, 0, spp3, stats=est)
            row[iname + "_segments_per_s"] = est.segments / (est.device_ms / 1e3)
            row[iname + "_frame_s"] = est.device_ms / 1e3
            row[iname + "_clocks"] = ck.summary()
        row["st_speedup_vs_pt"] = row["pt_frame_s"] / row["st_frame_s"]
        sweep.append(row)
    extra["c3_density_sweep"] = {"scene": f"bumpy sphere(4), 512x512 @ {spp3} spp (full frames), NEE",
                                 "rows": sweep}
    # FP64 parity mode on the bench scene (one 1-spp slab of the 1080p frame)
    r.upload_scene(scene)
    r.set_precision("f64")
    try:
        r.render_film(sb.ST, FRAME_SPP, 1, True, 0, 1)  # warm-up
        est = abi.PathStats()
        with ClockSampler(nvml_index(local)) as ck:
            r.render_film(sb.ST, FRAME_SPP, 1, True, 1, 2, stats=est)
        extra["c5_f64_parity_mode"] = {"slab": "1920x1080 @ 1 spp, ST+NEE, FP64 parity build (-fmad=false)",
                                       "segments_per_s": est.segments / (est.device_ms / 1e3),
                                       "slab_ms": est.device_ms, "clocks": ck.summary()}
    finally:
        r.set_precision("f32")
    # CVAE training (row f3): the desk-scale weights job, 3 kinds concurrently
    ds, _ = r.generate_dataset(200000, seed=7)
    r.train_models(ds[:5000], dataset_seed=7, epochs=1)  # warm-up
    t0 = time.perf_counter()
    _, tst = r.train_models(ds, dataset_seed=7, epochs=20, seed=1)
    tw = time.perf_counter() - t0
    dev_s = max(x.device_ms for x in tst) / 1e3  # the three kinds run concurrently
    extra["cvae_training"] = {"sample_passes_per_s": sum(x.sample_passes for x in tst) / dev_s,
                              "device_s": dev_s, "wall_s": tw,
                              "us_per_batch": [x.device_ms * 1e3 / max(x.steps, 1) for x in tst],
                              "workload": "train_model x3 kinds concurrently, 2e5 samples, 20 epochs, "
                                          "batch 512 (desk-scale weights job)"}
    return extra


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--spp-per-step", type=int, default=32)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--ref-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--no-frame", action="store_true")
    ap.add_argument("--quick-extra", action="store_true", help="extras on reduced sizes (development)")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args.gpus)
    world, rank, local = dist_env()
    if args.impl == "reference":
        bench_reference(args, world, rank)
    else:
        bench_ours(args, world, rank, local)
    return 0


if __name__ == "__main__":
    sys.exit(main())
