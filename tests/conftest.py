"""Shared fixtures.  `gpu`-marked tests need a B200 (run through gpurun);
everything else runs on the CPU-only build box."""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: large-size GPU parity cases")


def golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def golden_names(prefix: str) -> list[str]:
    return sorted(p.stem for p in GOLDEN.glob(f"{prefix}*.npz"))


def make_fuzzy(seed, n, dims, weighted=False):
    """conftest.make_fuzzy_ensemble draws (/root/reference/pkg/tests/conftest.py:20-29)."""
    rng = np.random.default_rng(seed)
    cells = int(np.prod(dims))
    w = rng.uniform(0.5, 2.0, size=cells) if weighted else None
    U = np.stack([rng.uniform(0.0, 1.0, size=cells).astype(np.float32) for _ in range(n)])
    return U, w


def make_binary(seed, n, dims, weighted=False):
    """conftest.make_binary_ensemble draws (/root/reference/pkg/tests/conftest.py:32-42)."""
    rng = np.random.default_rng(seed)
    cells = int(np.prod(dims))
    w = rng.uniform(0.5, 2.0, size=cells) if weighted else None
    rows = []
    for _ in range(n):
        d = rng.uniform(0.2, 0.8)
        rows.append((rng.uniform(0.0, 1.0, size=cells) < d).astype(np.float32))
    return np.stack(rows), w


# nested_trio (/root/reference/pkg/tests/conftest.py:45-58)
TRIO = np.array([[1, 1, 1, 0], [0, 1, 1, 0], [0, 1, 0, 0]], dtype=np.float32)
TRIO_IDS = ["c0", "c1", "c2"]


@pytest.fixture
def gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return torch.device("cuda", 0)
