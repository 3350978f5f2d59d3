"""Hardware check of the tcgen05 operand layouts (tests/native/umma_probe.cu)."""
import shutil
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu


def test_umma_layout_probe(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    src = Path(__file__).parent / "native" / "umma_probe.cu"
    exe = tmp_path / "probe"
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17", "-o", str(exe),
                    str(src)], check=True, capture_output=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120).stdout
    lines = [l for l in out.splitlines() if l.startswith("PROBE")]
    ok = {l.split("cuda=")[0].strip(): "maxerr=0 " in l for l in lines}
    assert ok["PROBE SS A-Kmajor"] and ok["PROBE SS A-MNmajor sbo=528"] and ok["PROBE TS A-tmem"], out
