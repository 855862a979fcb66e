"""The C-ABI library loads and exports every symbol include/cbspmv.h declares (CPU only)."""
import os
import re
import subprocess

import paper_2605_18515_b200 as cb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "cbspmv.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cbspmv_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared()
    for n in ("cbspmv_build", "cbspmv_spmv", "cbspmv_destroy"):
        assert n in names


def test_library_exports_every_declared_symbol():
    lib = cb.lib()
    out = subprocess.run(["nm", "-D", "--defined-only", cb.LIB_PATH], capture_output=True, text=True, check=True)
    exported = set(re.findall(r"\bT (cbspmv_\w+)", out.stdout))
    for n in declared():
        assert n in exported, n
        assert hasattr(lib, n)
    assert cb.version() == 1


def test_status_strings_and_null_safety():
    L = cb.lib()
    assert L.cbspmv_status_string(0) == b"CBSPMV_OK"
    assert L.cbspmv_status_string(6) == b"CBSPMV_EUNSUPPORTED"
    assert L.cbspmv_destroy(None) == 0
    assert L.cbspmv_build(1, 1, 0, None, None, None, 0, None, None, None) == 1  # null out


def test_no_oracle_in_product_path():
    """The product package must not import or link the oracle (independence rule)."""
    pkg = os.path.join(ROOT, "paper_2605_18515_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "liboracle" not in txt and "oracle_" not in txt, f
    out = subprocess.run(["ldd", cb.LIB_PATH], capture_output=True, text=True)
    assert "oracle" not in out.stdout


def test_host_only_handle_refuses_device_calls():
    import numpy as np
    import synth
    h = cb.build(synth.fig1(), device=-1)
    st = cb.lib().cbspmv_spmv(h.raw, 8, 16, None)
    assert st == 6
    assert h.info["nb"] == 1
    cb.destroy(h)
    np.testing.assert_equal(h._raw, None)


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    """No fallback: without libcbspmv.so every entry point raises."""
    import pytest
    mod = cb
    monkeypatch.setattr(mod, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(mod, "_lib", None)
    with pytest.raises(RuntimeError):
        mod.lib()
    import synth
    with pytest.raises(RuntimeError):
        mod.build(synth.fig1(), device=-1)


def test_new_entry_points_validate_arguments_without_a_gpu():
    """cbspmv_spmv_host_batch and cbspmv_xchg_* reject bad arguments before touching CUDA."""
    import ctypes

    import numpy as np
    import synth
    L = cb.lib()
    h = cb.build(synth.fig1(), device=-1)
    xs = [np.zeros(16)]
    ys = [np.zeros(16)]
    xp = (ctypes.c_void_p * 1)(xs[0].ctypes.data)
    yp = (ctypes.c_void_p * 1)(ys[0].ctypes.data)
    assert L.cbspmv_spmv_host_batch(h.raw, xp, yp, 1, None) == 6  # host-only handle: EUNSUPPORTED
    assert L.cbspmv_spmv_host_batch(None, xp, yp, 1, None) == 1
    cb.destroy(h)
    out = ctypes.c_void_p()
    for n, dt, world, rank, dev in ((16, 0, 9, 0, 0), (16, 0, 2, 2, 0), (-1, 0, 1, 0, 0), (16, 7, 1, 0, 0),
                                    (16, 0, 0, 0, 0), (16, 0, 1, 0, -1)):
        assert L.cbspmv_xchg_create(n, dt, world, rank, dev, ctypes.byref(out)) == 1  # EINVAL
        assert out.value is None
    assert L.cbspmv_xchg_destroy(None) == 0
    assert L.cbspmv_xchg_base(None) is None and L.cbspmv_xchg_buffer(None, 0) is None
    assert L.cbspmv_xchg_publish(None, 0, 0, 1, 1, None) == 1
    assert L.cbspmv_xchg_wait(None, 1, None, 1.0, None) == 1
