"""Shared synthetic-input recipes for the tests (seeded numpy)."""
import numpy as np


def outlier_matrix(rows, cols, seed=0, body=1.0, channels=(), tokens=(), mag_c=123.5,
                   mag_t=605.8, occasional=0, mag_o=150.9):
    """Gaussian body + injected outlier channels/tokens (synth.cpp:36-95 recipe)."""
    rng = np.random.default_rng(seed)
    x = (rng.standard_normal((rows, cols)) * body).astype(np.float32)
    for t in tokens:
        x[t, :] = np.where(rng.random(cols) < 0.5, -mag_t, mag_t)
    for c in channels:
        x[:, c] = np.where(rng.random(rows) < 0.5, -mag_c, mag_c)
    for _ in range(occasional):
        x[rng.integers(rows), rng.integers(cols)] = mag_o * (1 if rng.random() < 0.5 else -1)
    return x


def bf16_round(x):
    """Round-to-nearest-even fp32 -> bf16 -> fp32 (numpy), as torch does."""
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16).to(torch.float32).numpy()


def rel_fro(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    d = np.linalg.norm(a - b)
    n = np.linalg.norm(b)
    return d / n if n > 0 else d
