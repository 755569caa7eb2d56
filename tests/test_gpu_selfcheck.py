"""Memory-safety and race checks of the fused kernel without compute-sanitizer
(closed on this pool): the self-checking build libndgi_checked.so (build.py
build_checked) traps on any out-of-bounds shared-memory index or global
read / write offset (NDGI_CHECKED) and inserts random per-warp delays at every
synchronisation point (NDGI_JITTER: CTA barriers, the per-warp __syncwarp
hand-offs of the F_uv chunk and the F_uvt windows, the MMA round trips).  Each
case (FULL8, TILES8 with 4-row strips / short strips / whole tiles, RGBA32F,
the windowed H profile, a border wider than half the core, h = 64, C = 256,
BC3, mixed BC7 modes) must run without a trap and produce output bit-identical
to the product build's: a missing barrier or a TMEM / smem aliasing race would
make the jittered schedule's output differ."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2604_12625_b200"))
import build as ndgi_build  # noqa: E402

import selfcheck_run  # noqa: E402


def test_checked_jittered_build_matches_product(tmp_path):
    lib = ndgi_build.build_checked()
    out = tmp_path / "checked.npz"
    env = dict(os.environ, NDGI_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "selfcheck_run.py"), str(out)], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    ref = tmp_path / "product.npz"
    selfcheck_run.run(str(ref))
    a, b = np.load(out), np.load(ref)
    assert sorted(a.files) == sorted(b.files)
    for k in a.files:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
