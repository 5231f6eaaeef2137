"""The tcgen05.mma + tensor-memory Gram pipeline of tools/microbench/
(profiles/r02_tcgen05_experiment.txt): it is not on the product path (it
measured slower than the mma.sync kernel), but it is kept compiling for
sm_100a -- with the Blackwell tensor instructions in its SASS -- and correct
on the device: descriptors, swizzle, tensor-memory layout and the hi/lo
accuracy are checked against a host fp64 computation."""
import os
import shutil
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tools", "microbench", "umma_gram.cu")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _build(out):
    cmd = [NVCC, "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-o", out, SRC]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


@pytest.mark.skipif(not os.path.exists(NVCC), reason="no nvcc")
def test_umma_microbench_compiles_with_tcgen05_sass(tmp_path):
    exe = str(tmp_path / "umma_gram")
    _build(exe)
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    sass = subprocess.run([cuobjdump, "-sass", exe], capture_output=True, text=True).stdout
    for mnemonic in ("UTCHMMA", "UTCBAR", "LDTM"):  # tcgen05.mma, tcgen05.commit, tcgen05.ld
        assert mnemonic in sass, mnemonic


@pytest.mark.gpu
def test_umma_gram_matches_host_reference(tmp_path):
    exe = str(tmp_path / "umma_gram")
    _build(exe)
    r = subprocess.run([exe, "check"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "checks failed: 0" in r.stdout
