"""generate_synthetic (reference trace.py:218-268): the host generator and the device one
(librsim rsim_synth_generate, csrc/rsim_synth.cuh) against fingerprints of the reference's own
generator (tests/golden/synth_golden.json, made by tools/make_synth_golden.py), and the
restated glibc log the device uses for expovariate against the C library's."""
import hashlib
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "synth_golden.json")))
NAMES = [k for k in GOLD if not k.startswith("_")]
COLS = ("request_id", "arrival_s", "in_tokens", "out_tokens", "class_key", "blk_off", "blocks")


def _spec(name):
    from paper_2603_15202_b200.trace import ClassSpec, SyntheticSpec
    dur, rate, classes, seed, bs = eval(GOLD[name]["spec"])
    return SyntheticSpec(dur, rate, tuple(ClassSpec(*c) for c in classes), seed=seed, block_size=bs)


def _check(trace, name):
    want = GOLD[name]
    assert len(trace) == want["n"]
    for col in COLS:
        got = hashlib.sha256(np.ascontiguousarray(getattr(trace, col)).tobytes()).hexdigest()
        assert got == want["sha256"][col], f"{name}: column {col} differs from the reference generator"


def _libm_path():
    out = subprocess.run(["gcc", "-print-file-name=libm.so.6"], capture_output=True, text=True).stdout.strip()
    return out if os.path.isabs(out) else "/lib/x86_64-linux-gnu/libm.so.6"


def test_glibc_log_restatement_matches_libm(tmp_path):
    """rsim_log.h's glibc_log, compiled for the host, returns the C library's log() bit for bit
    on 8M inputs (half of them the expovariate inputs 1 - k 2^-53)."""
    exe = tmp_path / "check"
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-o", str(exe),
                    os.path.join(ROOT, "tools", "check_glibc_log.c"), "-lm"], check=True)
    r = subprocess.run([str(exe), "8000000", "3"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout


def test_glibc_log_constants_are_this_libm(tmp_path):
    """The committed constants are the ones in this image's libm (the one CPython calls)."""
    out = tmp_path / "h.h"
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "extract_glibc_log.py"), _libm_path(), str(out)],
                   check=True, capture_output=True)
    have = open(os.path.join(ROOT, "paper_2603_15202_b200", "csrc", "rsim_glibc_log.h")).read().splitlines()[1:]
    assert out.read_text().splitlines()[1:] == have


@pytest.mark.parametrize("name", [n for n in NAMES if GOLD[n]["n"] <= 200_000])
def test_host_generator_matches_reference(name):
    from paper_2603_15202_b200.trace import generate_synthetic_packed
    _check(generate_synthetic_packed(_spec(name)), name)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_device_generator_matches_reference(name):
    from paper_2603_15202_b200.trace import generate_synthetic_device
    _check(generate_synthetic_device(_spec(name)), name)


@pytest.mark.gpu
def test_device_generator_equals_host_generator():
    from paper_2603_15202_b200.trace import ClassSpec, SyntheticSpec, generate_synthetic_device, \
        generate_synthetic_packed
    rng = np.random.default_rng(17)
    for trial in range(6):
        k = int(rng.integers(1, 12))
        w = rng.dirichlet(np.ones(k))
        w[-1] = 1.0 - w[:-1].sum()
        classes = tuple(ClassSpec(float(w[i]), int(rng.integers(0, 6)), (1, int(rng.integers(1, 9))),
                                  (1, int(rng.integers(1, 300)))) for i in range(k))
        spec = SyntheticSpec(float(rng.uniform(1, 300)), float(rng.uniform(1, 80)), classes,
                             seed=int(rng.integers(0, 2**63)), block_size=int(rng.integers(1, 33)))
        a, b = generate_synthetic_device(spec), generate_synthetic_packed(spec)
        for col in COLS:
            assert np.array_equal(getattr(a, col).view(np.uint64) if col == "arrival_s" else getattr(a, col),
                                  getattr(b, col).view(np.uint64) if col == "arrival_s" else getattr(b, col)), \
                (trial, col)


@pytest.mark.gpu
def test_device_generator_spec_errors():
    """Invalid specs fail like the reference's SyntheticSpec.validate (TraceError); the C entry
    point checks the same rules itself."""
    import ctypes as C
    from paper_2603_15202_b200 import _native
    from paper_2603_15202_b200.trace import ClassSpec, SyntheticSpec, TraceError, generate_synthetic_device
    with pytest.raises(TraceError):
        generate_synthetic_device(SyntheticSpec(10.0, 1.0, (ClassSpec(0.5, 1),)))
    L = _native.lib()
    arr = (_native.SynthClass * 1)(_native.SynthClass(1.0, 0, 0, 0, 1, 2))   # zero blocks per request
    g = C.c_void_p()
    st = L.rsim_synth_generate(C.cast(arr, C.c_void_p), 1, 10.0, 1.0, 0, 16, 0, C.byref(g), None, None)
    assert st == _native.E_TRACE and b"at least one block" in L.rsim_last_error(None)


@pytest.mark.gpu
def test_device_generator_rerun_when_arrivals_overflow(monkeypatch):
    """Arrival buffers sized one per class (RSIM_SYNTH_TIGHT) overflow: the generator counts,
    reruns the arrival pass with exact room, and still matches the reference."""
    from paper_2603_15202_b200.trace import generate_synthetic_device
    monkeypatch.setenv("RSIM_SYNTH_TIGHT", "1")
    for name in ("chat_cfg1", "many_classes", "sparse_short"):
        _check(generate_synthetic_device(_spec(name)), name)
