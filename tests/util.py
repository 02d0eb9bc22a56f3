"""Shared helpers for the tests (inputs, scenes, comparisons)."""
import numpy as np

GOLDEN = 0x9E3779B97F4A7C15
MASK = (1 << 64) - 1


def state_after(state: int, draws: int) -> int:
    """RandomStream state after `draws` next_u64 calls (rng.hpp:25-28)."""
    return (int(state) + draws * GOLDEN) & MASK


def draws_between(s0, s1, max_draws=2000):
    """Number of draws that advanced state s0 to s1 (-1 if none <= max_draws)."""
    s0, s1 = int(s0), int(s1)
    for k in range(max_draws + 1):
        if (s0 + k * GOLDEN) & MASK == s1:
            return k
    return -1


def step_batch_from_golden(g, oracle_mod):
    keys = g["step_keys"]
    states = np.array([oracle_mod.rng_init(*[int(x) for x in k]) for k in keys], dtype=np.uint64)
    return dict(sigma_t=g["step_sigma_t"], g=g["step_g"], phi=g["step_phi"], w_in=g["step_w_in"],
                center=g["step_center"], r_sphere=g["step_r"], with_event=g["step_with_event"],
                rng_state=states)


def random_step_batch(n, seed, oracle_mod, sigma_hi=200.0):
    rng = np.random.default_rng(seed)
    w = rng.normal(size=(n, 3))
    w /= np.linalg.norm(w, axis=1)[:, None]
    states = np.array([oracle_mod.rng_init(seed, 6, i, 0) for i in range(n)], dtype=np.uint64)
    return dict(sigma_t=rng.uniform(0, sigma_hi, n), g=rng.uniform(-0.95, 0.95, n),
                phi=1 - 10 ** rng.uniform(-5, -0.3, n), w_in=w, center=rng.normal(size=(n, 3)),
                r_sphere=rng.uniform(0.01, 1.5, n), with_event=(rng.uniform(size=n) < 0.7).astype(np.uint8),
                rng_state=states)


def copy_batch(b):
    return {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in b.items()}


def rel_close(a, b, rtol, atol):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.abs(a - b) <= atol + rtol * np.abs(b)
