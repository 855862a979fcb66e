"""§8(b) boundary conventions (SURVEY.md §8(b) "Indexing and pointers"): every device-vector
entry point rejects a wrong dtype, length or device instead of reading or writing out of bounds.

CPU tests: the binding's checks (they run before any device call).  GPU tests: each rejection
through the binding, and the C layer's own checks (device identity, memory type, allocation
range) reached with raw pointers that bypass the binding."""
import ctypes

import numpy as np
import pytest

import paper_2605_18515_b200 as cb
import synth


# ----------------------------------------------------------------------------- CPU
def _host_handle():
    return cb.build(synth.fig1(), device=-1)


def test_binding_rejects_cpu_tensors_before_the_call():
    import torch
    h = _host_handle()
    x = torch.zeros(16, dtype=torch.float64)
    y = torch.zeros(16, dtype=torch.float64)
    for f in (cb.spmv, cb.spmv_add):
        with pytest.raises(ValueError, match="CUDA tensor"):
            f(h, x, y)
    with pytest.raises(ValueError, match="CUDA tensor"):
        cb.spmv_scaled(h, x, torch.ones(1, dtype=torch.float64), y)
    with pytest.raises(ValueError, match="CUDA tensor"):
        cb.spmv_panel(h, 0, x, None, y, True)
    cb.destroy(h)


def test_binding_rejects_non_tensor_vectors():
    h = _host_handle()
    with pytest.raises(TypeError):
        cb.spmv(h, np.zeros(16), np.zeros(16))
    cb.destroy(h)


def test_sumsq_rejects_other_dtypes():
    import torch
    for dt in (torch.bfloat16, torch.float16, torch.int64):
        with pytest.raises(TypeError):
            cb.sumsq(torch.zeros(8, dtype=dt), torch.zeros(1, dtype=torch.float64))


def test_c_layer_rejects_raw_pointers_on_a_host_handle():
    # raw pointers bypass the binding: the C layer still refuses (EUNSUPPORTED: host-only handle)
    h = _host_handle()
    with pytest.raises(cb.CBSpMVError) as e:
        cb.spmv(h, 4096, 8192)
    assert e.value.status == 6
    cb.destroy(h)


# ----------------------------------------------------------------------------- GPU
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    return torch


def _cudart():
    for name in ("libcudart.so.12", "libcudart.so"):
        try:
            L = ctypes.CDLL(name)
            L.cudaMalloc.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_size_t]
            L.cudaFree.argtypes = [ctypes.c_void_p]
            return L
        except OSError:
            continue
    pytest.skip("libcudart not loadable")


@pytest.fixture(scope="module")
def dev_handle():
    torch = _gpu()
    A = synth.clustered(1 << 10)
    h = cb.build(A, device=0)
    h32 = cb.build(A, dtype="f32", device=0)
    yield A, h, h32, torch
    cb.destroy(h)
    cb.destroy(h32)


def _ok_xy(A, torch, dt=None):
    dt = dt or torch.float64
    return torch.ones(A.n, dtype=dt, device="cuda:0"), torch.zeros(A.m, dtype=dt, device="cuda:0")


@pytest.mark.gpu
def test_binding_rejects_wrong_dtype(dev_handle):
    A, h, h32, torch = dev_handle
    x, y = _ok_xy(A, torch)
    x32, y32 = _ok_xy(A, torch, torch.float32)
    with pytest.raises(TypeError, match="dtype"):
        cb.spmv(h, x32, y)      # float32 x on an f64 handle
    with pytest.raises(TypeError, match="dtype"):
        cb.spmv(h, x, y32)
    with pytest.raises(TypeError, match="dtype"):
        cb.spmv(h32, x, y32)    # float64 x on an f32 handle
    with pytest.raises(TypeError, match="dtype"):
        cb.spmv_scaled(h, x, torch.ones(1, dtype=torch.float32, device="cuda:0"), y)
    cb.spmv(h, x, y)            # the well-formed call still runs
    cb.spmv(h32, x32, y32)
    torch.cuda.synchronize()


@pytest.mark.gpu
def test_binding_rejects_short_vectors(dev_handle):
    A, h, _, torch = dev_handle
    x, y = _ok_xy(A, torch)
    with pytest.raises(ValueError, match="elements"):
        cb.spmv(h, x[:-1], y)
    with pytest.raises(ValueError, match="elements"):
        cb.spmv_add(h, x, y[: A.m - 16])
    with pytest.raises(ValueError, match="elements"):
        cb.spmv_panel(h, 0, x, None, y[:1], True)
    with pytest.raises(ValueError, match="elements"):
        cb.spmv_scaled(h, x, torch.ones(0, dtype=torch.float64, device="cuda:0"), y)


@pytest.mark.gpu
def test_binding_rejects_non_contiguous(dev_handle):
    A, h, _, torch = dev_handle
    x2 = torch.ones(2 * A.n, dtype=torch.float64, device="cuda:0")[::2]
    y = torch.zeros(A.m, dtype=torch.float64, device="cuda:0")
    with pytest.raises(ValueError, match="contiguous"):
        cb.spmv(h, x2, y)


@pytest.mark.gpu
def test_c_layer_rejects_host_memory(dev_handle):
    A, h, _, torch = dev_handle
    x, y = _ok_xy(A, torch)
    xh = torch.ones(A.n, dtype=torch.float64).pin_memory()
    yh = torch.zeros(A.m, dtype=torch.float64)  # pageable: not a CUDA pointer at all
    with pytest.raises(cb.CBSpMVError) as e:
        cb.spmv(h, xh.data_ptr(), y.data_ptr())
    assert e.value.status == 5 and "device memory" in str(e.value)
    with pytest.raises(cb.CBSpMVError) as e:
        cb.spmv(h, x.data_ptr(), yh.data_ptr())
    assert e.value.status == 5


@pytest.mark.gpu
def test_c_layer_rejects_an_allocation_shorter_than_the_vector(dev_handle):
    A, h, _, torch = dev_handle
    L = _cudart()
    small = ctypes.c_void_p()
    assert L.cudaMalloc(ctypes.byref(small), 8 * (A.n // 2)) == 0  # its own allocation: half of x
    try:
        y = torch.zeros(A.m, dtype=torch.float64, device="cuda:0")
        with pytest.raises(cb.CBSpMVError) as e:
            cb.spmv(h, small.value, y.data_ptr())
        assert e.value.status == 5 and "allocation ends" in str(e.value)
        with pytest.raises(cb.CBSpMVError) as e:   # y in the short allocation
            cb.spmv(h, y.data_ptr(), small.value)
        assert e.value.status == 5
        # sumsq: v longer than its allocation
        out = torch.zeros(1, dtype=torch.float64, device="cuda:0")
        st = cb.lib().cbspmv_sumsq(small.value, A.n, cb.F64, out.data_ptr(), 0, None)
        assert st == 5
    finally:
        L.cudaFree(small)


@pytest.mark.gpu
def test_c_layer_rejects_a_sumsq_pointer_off_device(dev_handle):
    A, h, _, torch = dev_handle
    x, y = _ok_xy(A, torch)
    ss_host = torch.ones(1, dtype=torch.float64)
    with pytest.raises(cb.CBSpMVError) as e:
        cb.spmv_scaled(h, x, ss_host.data_ptr(), y)
    assert e.value.status == 5


@pytest.mark.gpu
def test_binding_rejects_wrong_device_index(dev_handle):
    A, h, _, torch = dev_handle
    if torch.cuda.device_count() < 2:
        # one GPU: a handle that claims device 0 against a CPU tensor is the reachable mismatch
        with pytest.raises(ValueError, match="CUDA tensor"):
            cb.spmv(h, torch.ones(A.n, dtype=torch.float64), torch.zeros(A.m, dtype=torch.float64))
        return
    x = torch.ones(A.n, dtype=torch.float64, device="cuda:1")
    y = torch.zeros(A.m, dtype=torch.float64, device="cuda:1")
    with pytest.raises(ValueError, match="handle is on cuda:0"):
        cb.spmv(h, x, y)
    with pytest.raises(cb.CBSpMVError) as e:
        cb.spmv(h, x.data_ptr(), y.data_ptr())
    assert e.value.status == 5
