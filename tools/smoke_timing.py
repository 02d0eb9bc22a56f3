import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_03082_b200 as sb
r = sb.Renderer(0, "f32")
r.load_models_dir(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "models"))
P, T = sb.make_icosphere(3, 1.0)
scene = sb.c1_scene((P, T), 16, 16, sdf_resolution=32)
r.upload_scene(scene)
for i in range(3):
    t0 = time.perf_counter()
    img, stats = r.render(sb.ST, 4, seed=1, nee=True)
    print(os.environ.get("TAG"), "device_ms", round(stats.device_ms, 2), "wall_ms", round(1e3 * (time.perf_counter() - t0), 2), stats.segments)
