"""GPU: C++ host code (examples/cpp_gmres.cpp) drives the path through the C
ABI / blkorth::gpu adapter and reproduces the reference's config-1 counts."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
EXE = Path(__file__).resolve().parents[1] / "examples" / "cpp_gmres"


@pytest.mark.parametrize("scheme", [0, 1])
def test_cpp_gmres_config1(gpu, scheme):
    if not EXE.exists():
        pytest.skip("examples/cpp_gmres not built")
    out = subprocess.run([str(EXE), str(scheme)], capture_output=True, text=True, timeout=300).stdout
    assert "converged=1" in out and "restarts=10 iterations=600" in out and "total=581" in out, out
    assert "bcgs2 on the Krylov panel: cols=6" in out
