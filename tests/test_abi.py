"""The C-ABI library loads on a CPU-only host and exports every symbol include/dmsgm.h declares.

No compute calls are made here (no GPU); on a CPU-only host dmsgm_create must fail
cleanly with DMSGM_ECUDA rather than crash, and argument errors must be reported
before any device work.
"""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def built():
    from paper_1702_05156_b200 import build
    return build.build()


HEADERS = ("dmsgm.h", "dmsgm_klt.h")


def _declared(header=None):
    names = set()
    for h in ([header] if header else HEADERS):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(dmsgm_[a-z_]+)\s*\(", src))
    return sorted(names)


def test_every_header_is_checked():
    assert sorted(f for f in os.listdir(os.path.join(ROOT, "include")) if f.endswith(".h")) == sorted(HEADERS)


def test_header_exports(built):
    lib = ctypes.CDLL(built)
    names = _declared()
    assert len(names) >= 22, names
    for n in names:
        assert hasattr(lib, n), f"{n} declared in include/ but not exported"
    import paper_1702_05156_b200 as dm
    assert sorted(dm.EXPORTS) == _declared("dmsgm.h")
    assert sorted(dm.KLT_EXPORTS) == _declared("dmsgm_klt.h")


def test_symbols_are_c_linkage(built):
    out = os.popen(f"nm -D --defined-only {built}").read()
    for n in _declared():
        assert re.search(rf"\bT {n}$", out, re.M), n


def test_version_and_argument_errors(built):
    import paper_1702_05156_b200 as dm
    assert "sm_100a" in dm.version()
    lib = dm.lib()
    p = dm.Params().to_c()
    h = ctypes.c_void_p()
    # invalid block size -> EINVAL before any CUDA call
    assert lib.dmsgm_create(64, 48, 3, ctypes.byref(p), 0, ctypes.byref(h)) == dm.DMSGM_EINVAL
    assert b"block" in lib.dmsgm_last_error(None)
    assert lib.dmsgm_create(66, 48, 4, ctypes.byref(p), 0, ctypes.byref(h)) == dm.DMSGM_EINVAL
    bad = dm.Params(theta_s=0.0).to_c()
    assert lib.dmsgm_create(64, 48, 4, ctypes.byref(bad), 0, ctypes.byref(h)) == dm.DMSGM_EINVAL
    assert lib.dmsgm_create(64, 48, 4, None, 0, ctypes.byref(h)) == dm.DMSGM_EINVAL
    big = dm.Params(age_cap=2.0 ** 25).to_c()        # the kernel's 1/(age+1) needs age_cap <= 2^24
    assert lib.dmsgm_create(64, 48, 4, ctypes.byref(big), 0, ctypes.byref(h)) == dm.DMSGM_EINVAL
    assert b"age_cap" in lib.dmsgm_last_error(None)
    assert lib.dmsgm_step(None, None, 64, None, None, 64, None) == dm.DMSGM_EINVAL
    # include/dmsgm_klt.h: parameter errors before any CUDA call
    from paper_1702_05156_b200 import klt
    L = klt._setup(lib)
    for bad in (dm.KltParams(win=2), dm.KltParams(max_corners=5000), dm.KltParams(quality=0.0),
                dm.KltParams(max_level=6), dm.KltParams(min_distance=0.5), dm.KltParams(ransac_iters=0)):
        cp = bad.to_c()
        assert L.dmsgm_klt_create(640, 480, ctypes.byref(cp), 0, ctypes.byref(h)) == dm.DMSGM_EINVAL
    cp = dm.KltParams().to_c()
    assert L.dmsgm_klt_create(4, 480, ctypes.byref(cp), 0, ctypes.byref(h)) == dm.DMSGM_EINVAL
    assert L.dmsgm_klt_estimate(None, None, 64, None, 64, None, None, None) == dm.DMSGM_EINVAL


def test_no_gpu_fails_cleanly(built):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1702_05156_b200 as dm
    with pytest.raises(dm.DmsgmError) as ei:
        dm.Dmsgm(64, 48, 4, dm.Params())
    assert ei.value.code == dm.DMSGM_ECUDA


def test_binding_has_no_fallback():
    """The product package never imports the oracle or a CPU implementation."""
    pkg = os.path.join(ROOT, "paper_1702_05156_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"(import\s+oracle|from\s+oracle|dmsgm_oracle|oracle/)", txt), f


def test_build_from_clean_checkout(tmp_path):
    """`python -m paper_1702_05156_b200.build` works without a prebuilt library."""
    import shutil
    import subprocess
    import sys
    shutil.copytree(os.path.join(ROOT, "include"), tmp_path / "include")
    shutil.copytree(os.path.join(ROOT, "paper_1702_05156_b200"), tmp_path / "paper_1702_05156_b200",
                    ignore=shutil.ignore_patterns("*.so", "__pycache__"))
    subprocess.check_call([sys.executable, "-m", "paper_1702_05156_b200.build"], cwd=tmp_path, timeout=600)
    assert (tmp_path / "paper_1702_05156_b200" / "libdmsgm.so").exists()
