"""C-ABI boundary checks that need no GPU: the in-tree librsim.so loads,
exports every entry point include/rsim.h declares, and refuses to run
without an sm_100 device (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rsim.h")
LIB = os.path.join(ROOT, "paper_2603_15202_b200", "librsim.so")


def declared():
    text = open(HEADER).read()
    protos = re.findall(r"^(?:rsim_status|void|const char|int64_t)\s*\*?\s*(rsim_\w+)\s*\(", text, re.M)
    return sorted(set(protos))


def test_header_declares_entry_points():
    names = declared()
    assert "rsim_create" in names and "rsim_replay" in names and "rsim_route_one" in names


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        import __graft_entry__ as g
        g.build()
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s+(rsim_\w+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing
    from paper_2603_15202_b200 import _native
    assert set(_native.EXPORTED) <= exported
    lib = ctypes.CDLL(LIB)
    for n in declared():
        getattr(lib, n)


def test_sass_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2603_15202_b200 import _native
    from paper_2603_15202_b200.cluster import Sizing, native_config
    from paper_2603_15202_b200.config import ClusterConfig
    with pytest.raises(_native.RsimError) as ei:
        _native.Handle(native_config(ClusterConfig(n_instances=2), Sizing(64, 100)))
    assert ei.value.status == _native.E_CUDA


def test_io_library_exports_every_declared_symbol():
    """librsimio.so (trace codec) exports every entry point include/rsim_io.h declares."""
    hdr = open(os.path.join(ROOT, "include", "rsim_io.h")).read()
    names = sorted(set(re.findall(r"^(?:int|void|const char|int64_t)\s*\*?\s*(rsim_\w+)\s*\(", hdr, re.M)))
    assert "rsim_trace_parse_jsonl" in names and len(names) == 6
    lib_path = os.path.join(ROOT, "paper_2603_15202_b200", "librsimio.so")
    if not os.path.exists(lib_path):
        import __graft_entry__ as g
        g.build()
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s+(rsim_\w+)", out))
    assert not [n for n in names if n not in exported]
