import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

# (check, max err/tol) of every tolerance check; printed at session end so a
# GPU run shows how much margin each parity class has.
MARGINS = []


def pytest_terminal_summary(terminalreporter):
    if not MARGINS:
        return
    worst = {}
    for what, m in MARGINS:
        worst[what] = max(worst.get(what, 0.0), m)
    terminalreporter.write_line("parity margins (max err / tolerance, < 1 passes): " +
                                ", ".join(f"{k} {v:.3g}" for k, v in sorted(worst.items())))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libgvr_cuda.so")


def golden_names():
    return sorted(os.path.splitext(os.path.basename(p))[0] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


class Golden:
    """One golden vector file: inputs + reference outputs."""

    def __init__(self, name):
        self.name = name
        self.g = dict(np.load(os.path.join(GOLDEN, name + ".npz")))

    def __getitem__(self, k):
        return self.g[k]

    def __contains__(self, k):
        return k in self.g

    @property
    def scene(self):
        from paper_2205_15401_b200.types import GaussianScene

        return GaussianScene(self.g["centers"], self.g["inv_cov"], self.g["attr"], float(self.g["tau"]))

    @property
    def camera(self):
        from paper_2205_15401_b200.types import Camera

        c = self.g["camera"]
        return Camera(c[:9].reshape(3, 3), c[9:12], c[12], c[13], c[14], int(c[15]), int(c[16]))

    @property
    def cfg(self):
        from paper_2205_15401_b200.types import SelectionConfig

        return SelectionConfig(float(self.g["eta"]), int(self.g["k_prime"]), bool(self.g["coarse"]),
                               int(self.g["ds"]))

    @property
    def flags(self):
        from paper_2205_15401_b200.types import GradFlags

        return GradFlags(bool(self.g["through_transmittance"]), bool(self.g["through_density"]))


@pytest.fixture(params=golden_names())
def golden(request):
    return Golden(request.param)


@pytest.fixture(scope="session")
def ctx():
    import paper_2205_15401_b200 as gvr

    return gvr.default_context(0)


def assert_close_rel(actual, ref, rel=1e-4, abs_floor=1e-7, what=""):
    """Parity rule 2: |x - x_ref| <= rel |x_ref| + abs_floor."""
    actual = np.asarray(actual)
    ref = np.asarray(ref)
    err = np.abs(actual - ref)
    bad = err > rel * np.abs(ref) + abs_floor
    MARGINS.append((what, float((err / (rel * np.abs(ref) + abs_floor)).max()) if err.size else 0.0))
    assert not bad.any(), (f"{what}: {bad.sum()} / {bad.size} entries out of tolerance; worst |err| "
                           f"{err.max():.3e} at ref {ref.reshape(-1)[np.argmax(err)]:.6e}")


def assert_grad_close(actual, ref, rel=1e-4, floor=1e-3, what=""):
    """Parity rule 3: |g - g_ref| <= rel max(|g_ref|, floor max_k |g_ref|) per class."""
    actual = np.asarray(actual)
    ref = np.asarray(ref)
    scale = np.abs(ref).max() if ref.size else 0.0
    tol = rel * np.maximum(np.abs(ref), floor * scale)
    err = np.abs(actual - ref)
    bad = err > tol
    if scale == 0.0:
        bad = err > 0.0
    MARGINS.append((what, float((err / np.maximum(tol, 1e-300)).max()) if err.size else 0.0))
    assert not bad.any(), (f"{what}: {bad.sum()} / {bad.size} out of tolerance; worst rel to scale "
                           f"{(err / max(scale, 1e-300)).max():.3e} (class scale {scale:.3e})")
