"""The C-ABI library builds for sm_100a, loads, and exports every symbol include/lsgcpd.h declares;
the ctypes struct layouts match the C header (no compute calls — runs without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lsgcpd.h")


@pytest.fixture(scope="module")
def L():
    from paper_2103_15039_b200 import build
    build.build()
    import paper_2103_15039_b200 as pkg
    return pkg.lib()


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(lsgcpd_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    syms = declared_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(L, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_2103_15039_b200", "liblsgcpd.so")],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (lsgcpd_\w+)", out))
    assert set(syms) <= exported
    assert all(s.startswith("lsgcpd_") for s in exported)


def test_version_and_pure_host_queries(L):
    assert L.lsgcpd_version() == 10400
    assert L.lsgcpd_last_error() is not None
    # header + body + tensor-core section + slot section (original index -> Morton slot)
    assert L.lsgcpd_target_bytes(1000) == 256 + 1024 * 64 + (1024 // 64) * 10240 + 1024 * 4
    assert L.lsgcpd_target_bytes(0) == 256


def test_struct_layouts_match_header(tmp_path):
    import paper_2103_15039_b200 as pkg
    prog = tmp_path / "sizes.c"
    prog.write_text('#include "lsgcpd.h"\n#include <stdio.h>\n#include <stddef.h>\n'
                    'int main(void){printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(lsgcpd_prep_params),'
                    ' sizeof(lsgcpd_target_info), sizeof(lsgcpd_annotations), sizeof(lsgcpd_em_params),'
                    ' offsetof(lsgcpd_em_params, sigma2_init), offsetof(lsgcpd_target_info, n_degenerate));'
                    'printf("%zu %zu %zu\\n", offsetof(lsgcpd_em_params, eta), offsetof(lsgcpd_em_params, d_src_conf),'
                    ' offsetof(lsgcpd_em_params, group));'
                    'return 0;}\n')
    exe = tmp_path / "sizes"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(prog), "-o", str(exe)])
    got = [int(v) for v in subprocess.check_output([str(exe)]).split()]
    want = [ctypes.sizeof(pkg.PrepParams), ctypes.sizeof(pkg.TargetInfo), ctypes.sizeof(pkg.Annotations),
            ctypes.sizeof(pkg.EmParams), pkg.EmParams.sigma2_init.offset, pkg.TargetInfo.n_degenerate.offset,
            pkg.EmParams.eta.offset, pkg.EmParams.d_src_conf.offset, pkg.EmParams.group.offset]
    assert got == want


def test_sass_is_sm100a_with_tma_bulk_copies():
    so = os.path.join(ROOT, "paper_2103_15039_b200", "liblsgcpd.so")
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", so], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass           # cp.async.bulk (TMA bulk copy) in the E-step kernel
    assert "MUFU.EX2" in sass


def test_oracle_is_not_imported_by_the_product():
    pkgdir = os.path.join(ROOT, "paper_2103_15039_b200")
    for dirpath, _, files in os.walk(pkgdir):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).lower() or f == "__init__.py" and \
                    "import oracle" not in txt, f


def test_only_test_infrastructure_imports_the_oracle():
    # oracle/ is test infrastructure: outside tests/, only __graft_entry__.smoke() and bench.py (cpu_baseline,
    # --impl reference) may import it; tools/, synth/ and include/ never do
    pat = re.compile(r"^\s*(import oracle|from oracle\b)", re.M)
    for top in ("tools", "synth", "include", "examples"):
        for dirpath, _, files in os.walk(os.path.join(ROOT, top)):
            for f in files:
                if f.endswith((".py", ".c", ".h", ".sh")):
                    assert not pat.search(open(os.path.join(dirpath, f)).read()), os.path.join(dirpath, f)


def test_missing_library_fails_loudly(tmp_path):
    # no CPU fallback: without liblsgcpd.so the binding raises on first use
    code = ("import paper_2103_15039_b200 as p\n"
            "try:\n    p.lib()\nexcept ImportError as e:\n    print('raised', 'no CPU fallback' in str(e))\n")
    env = dict(os.environ, LSGCPD_LIB=str(tmp_path / "missing.so"))
    out = subprocess.run(["python", "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert out.stdout.strip() == "raised True", out.stdout + out.stderr
