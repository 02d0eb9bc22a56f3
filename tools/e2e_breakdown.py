"""Where the end-to-end (host-buffer API) step time goes on the bench's C5 slab:
scene upload, synchronous device-film render, synchronous host-film render (+ D2H and
host accumulation), vs the asynchronous steady state.  python tools/e2e_breakdown.py"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import bench
import paper_2011_03082_b200 as sb
from paper_2011_03082_b200 import abi

r = sb.Renderer(0, "f32")
r.load_models_dir(bench.MODELS)
scene = bench.build_scene_ours(sb)
r.upload_scene(scene)
n = 3 * 1920 * 1080
S = 32
dev = torch.zeros(2 * n, dtype=torch.float64, device="cuda")
film = sb.Film(1920, 1080, np.zeros(n), np.zeros(n), 0)

def t(f, k=3):
    out = []
    for i in range(k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f(i)
        torch.cuda.synchronize()
        out.append(1e3 * (time.perf_counter() - t0))
    return [round(x, 1) for x in out]

for i in range(2):
    r.render_film(sb.ST, 5000, 1, True, i * S, (i + 1) * S, film)
print("upload_scene ms", t(lambda i: r.upload_scene(scene)))
print("render sync device film ms", t(lambda i: r.render_device(sb.ST, 5000, (4 + i) * S, (5 + i) * S, 1, True,
                                                              dev.data_ptr(), dev.data_ptr() + 8 * n)))
print("render_film host ms", t(lambda i: r.render_film(sb.ST, 5000, 1, True, (8 + i) * S, (9 + i) * S, film)))
print("upload + render_film ms", t(lambda i: (r.upload_scene(scene), r.render_film(sb.ST, 5000, 1, True, (12 + i) * S, (13 + i) * S, film))))
def asyn(i):
    for k in range(8):
        r.render_device(sb.ST, 5000, (20 + 8 * i + k) * S, (21 + 8 * i + k) * S, 1, True, dev.data_ptr(),
                        dev.data_ptr() + 8 * n, asynchronous=True)
    r.read_stats()
print("8 async slabs ms", t(asyn, 2))
