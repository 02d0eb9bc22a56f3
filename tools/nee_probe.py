import sys; sys.path.insert(0, ".")
import paper_2011_03082_b200 as sb
r = sb.Renderer(0, "f32"); r.load_models_dir("tests/golden/models")
for a in [(10.0, 0.8, 0.9), (5.0, -0.5, 1.0), (20.0, 0.3, 0.95)]:
    for (w, R) in [(100000, 10), (100000, 100), (1000000, 10)]:
        for seed in (3, 4, 5):
            x = r.nee_identity(w, R, *a, light=(0.0, 2.0, 2.0), seed=seed)
            print(a, w, R, seed, x.full_mean, x.single_mean, (x.single_mean - x.full_mean) / x.full_mean, (x.single_mean - x.full_mean) / x.diff_stderr, flush=True)
