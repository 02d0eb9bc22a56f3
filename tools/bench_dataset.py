"""Config 4 throughput: CVAE training-data generation (BASELINE.json configs[3]: 1e8
random-walk photons in the unit sphere over sigma_t in [0,200], g in [-1,1]).

  python tools/bench_dataset.py [--n 10000000] [--precision f32] [--cpu-seconds 10]

Prints one JSON line: walks/s and events/s on the GPU (device-resident output, chunked),
the extrapolated time for 1e8 walks, and the reference CPU rate (oracle/_ref
generate_dataset on all host cores, bounded sample) when available.
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2011_03082_b200 as sb  # noqa: E402
from paper_2011_03082_b200 import abi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--precision", default="f32")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    a = ap.parse_args()
    import torch
    r = sb.Renderer(0, a.precision)
    chunk = min(a.n, 1 << 24)
    dev = torch.empty(chunk * 52, dtype=torch.uint8, device="cuda")
    st = abi.DatasetStats()
    # warm-up
    abi.check(abi.lib().sst_gpu_generate_dataset(r.h, 100000, 0.0, 200.0, -1.0, 1.0, 0, -5.0, -0.5, 7, 0,
                                                 C.c_void_p(dev.data_ptr()), abi.SST_PTR_DEVICE, None))
    t0 = time.perf_counter()
    for b in range(0, a.n, chunk):
        m = min(chunk, a.n - b)
        abi.check(abi.lib().sst_gpu_generate_dataset(r.h, m, 0.0, 200.0, -1.0, 1.0, 0, -5.0, -0.5, 7, b,
                                                     C.c_void_p(dev.data_ptr()), abi.SST_PTR_DEVICE,
                                                     C.byref(st)))
    wall = time.perf_counter() - t0
    line = {"config": "c4 dataset generation", "precision": a.precision, "walks": st.walks,
            "events": st.events, "replay_events": st.replay_events, "max_events": st.max_events,
            "device_s": st.device_ms / 1e3, "wall_s": wall,
            "walks_per_s": st.walks / (st.device_ms / 1e3), "events_per_s": st.events / (st.device_ms / 1e3),
            "time_1e8_walks_s": 1e8 / (st.walks / (st.device_ms / 1e3))}
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    try:
        import reflib
        if reflib.available() and a.cpu_seconds > 0:
            os.environ["SST_THREADS"] = str(os.cpu_count())
            n = 2000
            t = time.perf_counter()
            d = reflib.generate_dataset(n, seed=9)
            dt = time.perf_counter() - t
            n = int(max(2000, n * a.cpu_seconds / max(dt, 1e-3)))
            t = time.perf_counter()
            d = reflib.generate_dataset(n, seed=10)
            dt = time.perf_counter() - t
            line["cpu_reference"] = {"walks_per_s": n / dt, "events_per_s": float(d["n_events"].astype(np.float64).sum()) / dt,
                                     "cores": os.cpu_count(), "sample": f"{n} walks"}
            line["speedup_vs_cpu"] = line["walks_per_s"] / line["cpu_reference"]["walks_per_s"]
    except Exception as e:  # noqa: BLE001
        line["cpu_reference"] = {"error": str(e)}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
