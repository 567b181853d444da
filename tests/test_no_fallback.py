"""The product path has no CPU fallback: without a GPU, or without the CUDA library,
every call fails loudly instead of computing anything on the host."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="this check needs a machine without a GPU")
def test_context_without_gpu_raises():
    from paper_1802_05839_b200 import weather as W
    with pytest.raises(W.HftwError) as e:
        W.Context(W.GridConfig(nx=8, ny=8, nz=4))
    assert "ECUDA" in str(e.value) or "cuda" in str(e.value).lower()


@pytest.mark.skipif(_has_gpu(), reason="this check needs a machine without a GPU")
def test_run_reference_without_gpu_raises():
    from paper_1802_05839_b200 import weather as W
    with pytest.raises(W.HftwError):
        W.run_reference(W.GridConfig(nx=8, ny=8, nz=4), 1)


def test_missing_library_is_an_error():
    """A library path that does not exist is an import-time error, not a fallback."""
    code = ("from paper_1802_05839_b200 import _lib\n"
            "try:\n"
            "    _lib.lib()\n"
            "except OSError as e:\n"
            "    print('OSError')\n")
    env = dict(os.environ, HFTW_LIBRARY=os.path.join(ROOT, "no_such_dir", "libhftw.so"))
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True,
                         text=True, timeout=600)
    assert "OSError" in out.stdout, out.stdout + out.stderr
