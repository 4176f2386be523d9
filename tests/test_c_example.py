"""examples/register_c.c: the C ABI used from plain C (CUDA runtime for device memory, no Python or torch).
It compiles against include/lsgcpd.h on the CPU; on a GPU it recovers a noiseless transform exactly."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    from paper_2103_15039_b200 import build
    build.build()
    out = tmp_path_factory.mktemp("cex") / "register_c"
    libdir = os.path.join(ROOT, "paper_2103_15039_b200")
    subprocess.check_call(["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           "-I", os.path.join(CUDA, "include"), os.path.join(ROOT, "examples", "register_c.c"),
                           "-L", libdir, "-llsgcpd", "-L", os.path.join(CUDA, "lib64"), "-lcudart", "-lm",
                           f"-Wl,-rpath,{libdir}", "-o", str(out)])
    return str(out)


def test_c_example_compiles_and_links(exe):
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_c_example_recovers_the_transform(exe):
    p = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "rotation error" in p.stdout
