#!/usr/bin/env python
"""Benchmark of the north-star path: CVAE sphere tracing (SDF safe radius -> CVAE
sphere step -> NEE -> continue/exit) on the config-5 teaser scene of BASELINE.json
(1920x1080, four media sigma_t = 20/40/80/160, g = 0.8), one JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--spp-per-step S] [--impl ours|reference]

A step = one sample slab of S spp over every pixel and channel of the 1080p frame
(3 * 1920 * 1080 * S light paths) on each rank; ranks render disjoint sample slabs
(weak scaling) and the film (FP64 sum and sum of squares) is reduced to rank 0 with
NCCL at the end of the timed region. value = light-path segments (sphere steps +
delta-tracking events, counted on the device) of all ranks / max-over-ranks time.

--impl reference runs the reference's own CPU implementation (oracle/_ref: the
reference sources + the reference-composed integrator) on the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
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
#   wf_logic  HBM: per slot visit the path state it must read (x,L 16 + w,r 16 + rng 8 +
#             meta 16 + flight 4 + trace position 4 = 64 B), write back (60 B) and its
#             live-list entry (4 B); per flight it sends to the trace kernel the 36 B ray
#             record + trace position (4 B) + the 12 B result it reads back next pass
#             (traversals minus the one shared camera ray per pixel-sample); per fresh path
#             the camera-ray result and direction (28 B); per delta-tracking event its NEE
#             record + queue entry (36 B); per sphere request a queue entry (4 B).
#   wf_trace  FP32: per interior node 2 slab tests = 12 FFMA + 12 min/max = 36 FLOP;
#             per Moller-Trumbore test 51 FLOP (2 cross, 4 dot, rcp, 3 mul, 3 sub).
#   wf_shadow FP32: 51 FLOP per light-grid triangle test.
#   wf_sphere FP32: decoder MLP FLOPs 2*(112 nL + 480 nP + 640 nE).
NODE_FLOP, TRI_FLOP = 36.0, 51.0
LOGIC_BYTES_PER_SLOT, LOGIC_BYTES_PER_FLIGHT, LOGIC_BYTES_PER_FRESH = 128.0, 52.0, 28.0
NEE_RECORD_BYTES, SPHERE_QUEUE_BYTES = 36.0, 4.0


def logic_bytes(k):
    """Algorithmic HBM bytes of the logic kernel over a measured slab (device counters)."""
    flights = max(0.0, float(k.traversals) - float(k.paths) / 3.0)
    return (LOGIC_BYTES_PER_SLOT * k.wavefront_slot_visits + LOGIC_BYTES_PER_FLIGHT * flights
            + LOGIC_BYTES_PER_FRESH * k.paths + NEE_RECORD_BYTES * k.pt_events
            + SPHERE_QUEUE_BYTES * k.sphere_steps)


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during the timed region."""
    NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
             0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
             0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz, self.ok = [], set(), None, False
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


def cpu_reference_rate(seconds: float, seed: int = 99, threads: int | None = None):
    """Times the reference CPU path (oracle/_ref) on a bounded random sample of the
    workload's light paths. Returns (segments/s, info)."""
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
        pix = rng.integers(0, W_FRAME * H_FRAME, n)
        smp = rng.integers(0, FRAME_SPP, n)
        ch = rng.integers(0, 3, n)
        st = abi.PathStats()
        t0 = time.perf_counter()
        rs.trace_paths(models, 1, 1, 1, pix, smp, ch, st)
        return time.perf_counter() - t0, st

    dt, st = run(4000)  # calibration
    rate_paths = 4000 / max(dt, 1e-6)
    n = int(max(4000, rate_paths * seconds))
    return run, n, threads


def bench_reference(args, world, rank):
    if rank != 0:
        return
    import platform
    run, n, threads = cpu_reference_rate(args.ref_seconds)
    for _ in range(args.warmup):
        run(max(1000, n // 10))
    tot_seg = 0
    tot_t = 0.0
    for _ in range(args.steps):
        dt, st = run(n)
        tot_seg += st.segments
        tot_t += dt
    value = tot_seg / tot_t
    cpu = platform.processor() or platform.machine()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "segments/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": DATA, "config": {"workload": WORKLOAD, "paths_per_step": n,
                                 "sample": f"{n} uniformly random (pixel, sample, channel) paths of the frame per step"},
        "cpu_baseline": {"value": value, "unit": "segments/s", "cores": threads, "kind": "reference",
                         "sample": f"{n} random light paths of the 1080p frame per step, {args.steps} steps",
                         "cpu": cpu},
        "e2e": {"value": value, "unit": "segments/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def load_traffic():
    p = os.path.join(PROFILES, "traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:  # noqa: BLE001
            return None
    return None


def bench_ours(args, world, rank, local):
    import torch

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
    stream = torch.cuda.ExternalStream(r.stream)
    n_pix = W_FRAME * H_FRAME
    S = args.spp_per_step
    total_steps = args.warmup + args.steps
    if (total_steps + 1) * world * S > FRAME_SPP:
        raise SystemExit("spp budget exceeds the 5000-spp frame")
    # FFMA roofline denominator (measured once, before the timed region)
    peak_lib = C.CDLL(os.path.join(ROOT, "paper_2011_03082_b200", "libsst_peak.so"))
    peak_lib.sst_peak_ffma_tflops.restype = C.c_double
    peak_lib.sst_peak_ffma_tflops.argtypes = [C.c_int, C.c_int]
    fp32_peak = peak_lib.sst_peak_ffma_tflops(local, 5)
    with torch.cuda.stream(stream):
        fsum = torch.zeros(3 * n_pix, dtype=torch.float64, device="cuda")
        fsq = torch.zeros(3 * n_pix, dtype=torch.float64, device="cuda")
        flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > L2

    def slab(step):
        s0 = (step * world + rank) * S
        return s0, s0 + S

    def one(step):
        with torch.cuda.stream(stream):
            flush.zero_()  # evict L2 between steps (inputs are L2-resident by design)
        s0, s1 = slab(step)
        # asynchronous enqueue: consecutive slabs pipeline on the context's streams
        r.render_device(sb.ST, FRAME_SPP, s0, s1, 1, True, fsum.data_ptr(), fsq.data_ptr(),
                        asynchronous=True)

    for i in range(args.warmup):
        one(i)
    r.read_stats()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(nvml_index(local)) as clocks:
        ev0.record(stream)
        for i in range(args.steps):
            one(args.warmup + i)
        stats = r.read_stats()  # joins the pipeline (device-side) and synchronises
        if dist:
            with torch.cuda.stream(stream):
                dist.reduce(fsum, dst=0)
                dist.reduce(fsq, dst=0)
        ev1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    seg = float(stats.segments)
    flops = mlp_flops(stats.decodes_length, stats.decodes_path, stats.decodes_event)
    dev_ms = stats.device_ms
    if dist:
        t = torch.tensor([ms, dev_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, dev_ms_max = t.tolist()
        s = torch.tensor([seg, flops, float(stats.paths), float(stats.sphere_steps),
                          float(stats.pt_events)], dtype=torch.float64, device="cuda")
        dist.all_reduce(s)
        seg_all, flops_all, paths_all, sphere_all, events_all = s.tolist()
    else:
        seg_all, flops_all, paths_all = seg, flops, float(stats.paths)
        sphere_all, events_all = float(stats.sphere_steps), float(stats.pt_events)
    value = seg_all / (ms / 1e3)
    ms_step = ms / args.steps
    # dominant kernel: the persistent trace kernel (plus the tiny film sum) of this rank
    achieved = flops / (dev_ms / 1e3) / 1e12
    traffic = load_traffic()
    hbm_bytes = paths_all * 8.0 + args.steps * world * 3 * n_pix * 32.0

    # ---- per-kernel roofline: one more slab with every launch bracketed by CUDA events
    # on its own stream (synchronous per iteration, so outside the timed region)
    hbm_peak = 6551.7
    try:
        hbm_peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:  # noqa: BLE001
        pass
    r.kernel_timing(True)
    kst = abi.PathStats()
    s0k = (args.warmup + args.steps) * world * S + rank * S
    r.render_device(sb.ST, FRAME_SPP, s0k, s0k + S, 1, True, fsum.data_ptr(), fsq.data_ptr(), stats=kst)
    kt = r.kernel_timing(False)
    tri_trace = kst.triangle_tests - kst.shadow_triangle_tests
    kdef = {
        "wf_logic": ("hbm", logic_bytes(kst) / 1e9,
                     hbm_peak, "GB/s"),
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

    # ---- e2e: the public host-buffer API per step (scene upload + render + film D2H)
    e2e = None
    if not args.no_e2e:
        film = sb.Film(W_FRAME, H_FRAME, np.zeros(3 * n_pix), np.zeros(3 * n_pix), 0)
        est = abi.PathStats()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        t_up = 0.0
        for i in range(args.steps):
            ta = time.perf_counter()
            r.upload_scene(scene)
            t_up += time.perf_counter() - ta
            s0, s1 = slab(args.warmup + i)
            r.render_film(sb.ST, FRAME_SPP, 1, True, s0, s1, film, est)
        t_e2e = time.perf_counter() - t0
        if os.environ.get("SST_BENCH_VERBOSE"):
            print(f"e2e: {t_e2e:.3f} s total, upload {t_up:.3f} s, device {est.device_ms / 1e3:.3f} s",
                  file=sys.stderr)
        e_seg = float(est.segments)
        if dist:
            t = torch.tensor([t_e2e], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t_e2e = t.item()
            t = torch.tensor([e_seg], dtype=torch.float64, device="cuda")
            dist.all_reduce(t)
            e_seg = t.item()
        e2e = {"value": e_seg / t_e2e, "unit": "segments/s",
               "h2d_bytes_per_step": int(info["h2d_bytes"]),
               "d2h_bytes_per_step": int(2 * 3 * n_pix * 8),
               "path": "sst_gpu_upload_scene + sst_gpu_render(SST_PTR_HOST) per step"}

    # ---- secondary configs (rank 0, single GPU work; not the headline metric)
    extra = None
    if rank == 0 and not args.no_extra:
        extra = {}
        mesh = sb.make_icosphere(3, 1.0)
        for name, integ in (("c1_st_nee", sb.ST), ("c2_pt_nee", sb.PT)):
            r.upload_scene(sb.c1_scene(mesh, 256, 256))
            r.render_film(integ, 64, 1, True, 0, 8)  # warm-up
            est = abi.PathStats()
            r.render_film(integ, 64, 1, True, 0, 64, stats=est)
            extra[name] = {"frame": "256x256 @ 64 spp", "frame_ms": est.device_ms,
                           "segments_per_s": est.segments / (est.device_ms / 1e3),
                           "segments_per_path": est.segments / est.paths}
        dst = abi.DatasetStats()
        out, _ = r.generate_dataset(200000, seed=7)  # warm-up
        dst = abi.DatasetStats()
        r.generate_dataset(8000000, seed=7, first_index=200000, stats=dst)
        extra["c4_dataset"] = {"walks_per_s": dst.walks / (dst.device_ms / 1e3),
                               "events_per_s": dst.events / (dst.device_ms / 1e3),
                               "time_1e8_walks_s": 1e8 / (dst.walks / (dst.device_ms / 1e3)),
                               "sample": "8e6 walks, sigma_t U[0,200], g U[-1,1], phi 1-10^U[-5,-0.5]"}
        # config 3: density-doubling sweep on the SDF-boundary bumpy-sphere scene (512x512)
        bumpy = sb.make_bumpy_sphere(4, 1.0, 0.2, 3.0)
        sweep = []
        for sig in (10.0, 40.0, 160.0):
            r.upload_scene(sb.c3_scene(bumpy, sig))
            row = {"sigma_t": sig}
            for iname, integ in (("st", sb.ST), ("pt", sb.PT)):
                r.render_film(integ, 1000, 1, True, 0, 1)  # warm-up
                est = abi.PathStats()
                r.render_film(integ, 1000, 1, True, 1, 9, stats=est)
                row[iname + "_segments_per_s"] = est.segments / (est.device_ms / 1e3)
                row[iname + "_frame_1000spp_s"] = est.device_ms / 8
            row["st_speedup_vs_pt"] = row["pt_frame_1000spp_s"] / row["st_frame_1000spp_s"]
            sweep.append(row)
        extra["c3_density_sweep"] = {"scene": "bumpy sphere(4), 512x512, NEE, 8 spp measured", "rows": sweep}
        # CVAE training (row f3): the desk-scale weights job, 3 kinds concurrently
        r.train_models(out[:5000], dataset_seed=7, epochs=1)  # warm-up
        t0 = time.perf_counter()
        _, tst = r.train_models(out, dataset_seed=7, epochs=20, seed=1)
        tw = time.perf_counter() - t0
        dev_s = max(x.device_ms for x in tst) / 1e3  # the three kinds run concurrently
        extra["cvae_training"] = {"sample_passes_per_s": sum(x.sample_passes for x in tst) / dev_s,
                                  "device_s": dev_s, "wall_s": tw,
                                  "us_per_batch": [x.device_ms * 1e3 / max(x.steps, 1) for x in tst],
                                  "workload": "train_model x3 kinds concurrently, 2e5 samples, 20 epochs, "
                                              "batch 512 (desk-scale weights job)"}
        r.upload_scene(scene)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        run, n, threads = cpu_reference_rate(args.ref_seconds / 2)
        dt, st = run(n)
        cpu = {"value": st.segments / dt, "unit": "segments/s", "cores": threads, "kind": "reference",
               "sample": f"{n} uniformly random (pixel, sample, channel) light paths of the 1080p frame "
                         f"({st.segments} segments, {dt:.1f} s), reference sources + reference-composed integrator"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "segments/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": DATA,
            "config": {
                "workload": WORKLOAD, "spp_per_step_per_gpu": S, "paths_per_step": int(paths_all / args.steps),
                "frame_spp": FRAME_SPP,
                "frame_time_s_extrapolated": ms_step / 1e3 * FRAME_SPP / (S * world),
                "sphere_steps": int(sphere_all), "pt_events": int(events_all),
                "l2": "flushed between steps by a 256 MB device write (scene is L2-resident by design)",
                "parallelism": f"sample slabs per rank x{world}" + (" + NCCL film reduce" if world > 1 else ""),
                "bvh_nodes": info["bvh_nodes"], "triangles": info["triangles"],
                "paths_per_s": paths_all / (ms / 1e3),
            },
            "roofline": {
                "bound": kernels[dominant]["bound"] if dominant else None,
                "achieved": kernels[dominant]["achieved"] if dominant else None,
                "peak": kernels[dominant]["peak"] if dominant else None,
                "unit": kernels[dominant]["unit"] if dominant else None,
                "frac": kernels[dominant]["frac"] if dominant else None,
                "traffic": (traffic or {}).get("kernels", {}).get(dominant, {}).get("dram_bytes_per_launch"),
                "kernel": f"k_{dominant} (wavefront)" if dominant else None,
                "share_of_kernel_time": kernels[dominant]["share"] if dominant else None,
                "achieved_def": "algorithmic work of the measured slab (device counters; bench.py NODE_FLOP/TRI_FLOP/"
                                "LOGIC_BYTES_PER_SLOT) / summed CUDA-event duration of that kernel's launches on "
                                "their stream (one extra slab after the timed region)",
                "peak_source": f"HBM: MEASURED_PEAKS.json hbm_gbs; FP32: measured FFMA throughput (csrc/peak.cu) "
                               f"{fp32_peak:.1f} TFLOP/s on this GPU (MEASURED_PEAKS.json has no FP32 figure)",
                "kernels": kernels,
                "decoder_flops": {"achieved": achieved, "unit": "TFLOP/s", "frac": achieved / fp32_peak if fp32_peak else None,
                                  "def": "decoder MLP FLOPs only / whole render device time (SURVEY §8d)"},
                "hbm_film": {"algorithmic_bytes_per_s": hbm_bytes / (ms / 1e3),
                             "frac_of_measured": hbm_bytes / (ms / 1e3) / (hbm_peak * 1e9),
                             "def": "per path 4 B radiance write + 4 B film read; film 2x8 B RMW per pixel-channel per slab"},
            },
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


def main():
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
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    world, rank, local = dist_env()
    if args.impl == "reference":
        bench_reference(args, world, rank)
    else:
        bench_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
