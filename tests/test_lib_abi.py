"""CPU-side checks of the C-ABI library: it builds, loads, and exports every symbol that
include/voxcap.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2004_02609_b200 as vc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    hdr = open(os.path.join(ROOT, "include", "voxcap.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(vc_[a-z_0-9]+)\s*\(", hdr)))


@pytest.fixture(scope="module")
def libpath():
    if not os.path.exists(vc.lib_path()):
        from paper_2004_02609_b200.build import build
        build()
    return vc.lib_path()


def test_header_matches_binding():
    assert sorted(vc.EXPORTS) == _declared()


def test_library_exports_every_declared_symbol(libpath):
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True,
                         text=True).stdout
    syms = set(re.findall(r"\b(vc_[a-z_0-9]+)\b", out))
    missing = [s for s in _declared() if s not in syms]
    assert not missing, missing
    lib = ctypes.CDLL(libpath)
    for s in _declared():
        assert hasattr(lib, s)


def test_library_is_sm100a(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_version_and_no_device_behaviour(libpath):
    lib = vc.load_library()
    assert b"sm_100a" in lib.vc_version()
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    ctx = ctypes.c_void_p()
    st = lib.vc_create(ctypes.byref(ctx), 0, None)
    assert st != 0  # fails loudly without a device: no CPU fallback
    with pytest.raises(vc.VoxCapError):
        vc.VoxCap(0)


def test_product_never_imports_oracle():
    """The product package shares no code with oracle/ (DESIGN.md §Oracle)."""
    pkg = os.path.join(ROOT, "paper_2004_02609_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f), errors="ignore").read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", src, re.M), f
                assert "kernels_q" not in src, f


def test_struct_layouts_match_header(tmp_path):
    """The ctypes mirrors of the option / info / stats structs have the sizes and field offsets
    the C compiler gives the header's definitions (a field added on one side only would shift
    every later field)."""
    import paper_2004_02609_b200 as m
    checks = {"vc_build_opts": m.BuildOpts, "vc_solve_opts": m.SolveOpts,
              "vc_solve_info": m.SolveInfo, "vc_stats": m.Stats}
    lines = ['#include <stddef.h>', '#include <stdio.h>', '#include "voxcap.h"', "int main(void) {"]
    for cname, cls in checks.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    cuda_inc = "/usr/local/cuda/include"
    r = subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-I", cuda_inc, str(src), "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {}
    for ln in out:
        if ln:
            a, b, c = ln.split()
            got[(a, b)] = int(c)
    for cname, cls in checks.items():
        assert got[(cname, "size")] == ctypes.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert got[(cname, fname)] == getattr(cls, fname).offset, (cname, fname)
