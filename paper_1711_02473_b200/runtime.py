"""ctypes binding of libsfk.so and the batched evaluation API.

Reference tier 2 of the boundary: per-cell execution is
the emitted C function driven by the caller's cell loop
(scheduling.py:731-735), or ``interpreter.run_kernel(program, inputs)``
(interpreter.py:279-378) in Python.  The drop-in here is

    evaluate_batched(plan, {"coords": (C, 24), "w0": (C, nd), ...}) -> (C, size)

which validates exactly like ``run_kernel`` (missing argument ->
``UnboundVariable``, wrong per-cell size -> ``ShapeMismatch``,
interpreter.py:291-299) and then makes ONE ``sfk_eval`` call: device
tensors run stream-ordered on the current torch stream; numpy (host) arrays
go through ``sfk_eval_host`` (pipelined H2D / compute / D2H).  There is no
CPU fallback: without a GPU or without libsfk.so every call raises.
"""

from __future__ import annotations

import contextlib
import ctypes
import os
import threading

import numpy as np

from .errors import NativeError, ShapeMismatch, UnboundVariable

__all__ = ["load_library", "evaluate_batched", "evaluate_batched_pair", "set_option",
           "get_option",
           "evaluate_host", "sum_squares", "launch_count", "fp64_peak",
           "device_info", "native_plan", "EXPORTED_SYMBOLS", "Mesh"]

_LIB = None
_LOCK = threading.Lock()
_dp = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p

EXPORTED_SYMBOLS = (
    "sfk_abi_version", "sfk_plan_create", "sfk_plan_destroy", "sfk_plan_sizes",
    "sfk_eval", "sfk_eval_pair", "sfk_eval_host", "sfk_sum_squares",
    "sfk_launch_count", "sfk_last_error", "sfk_device_info", "sfk_fp64_peak",
    "sfk_eval_gather_scatter", "sfk_program_create", "sfk_program_destroy",
    "sfk_program_sizes", "sfk_program_config", "sfk_program_text", "sfk_program_eval",
    "sfk_csr_create", "sfk_csr_info", "sfk_csr_destroy", "sfk_assemble_csr",
    "sfk_csr_entry_map", "sfk_eval_global", "sfk_eval_host_async", "sfk_host_wait",
    "sfk_csr_insert", "sfk_set_option", "sfk_get_option",
    "sfk_kernel_available", "sfk_mesh_create", "sfk_mesh_upload", "sfk_mesh_coords",
    "sfk_mesh_destroy", "sfk_eval_host_mesh",
)
ABI_VERSION = 1
SUM_WORKSPACE = 1024


def library_path():
    """In-tree libsfk.so; SFK_LIBRARY overrides the path (A/B runs of two
    builds of the same ABI)."""
    return os.environ.get("SFK_LIBRARY") or os.path.join(
        os.path.dirname(os.path.abspath(__file__)), "libsfk.so")


def _declare(lib):
    i64 = ctypes.c_int64
    ci = ctypes.c_int
    lib.sfk_abi_version.restype = ci
    lib.sfk_plan_create.argtypes = [ci, ci, ci, ci, ci, ci, _dp, _dp, _dp, _dp,
                                    _dp, _dp, _dp, ci, ctypes.POINTER(_vp)]
    lib.sfk_plan_create.restype = ci
    lib.sfk_plan_destroy.argtypes = [_vp]
    lib.sfk_plan_destroy.restype = ci
    lib.sfk_plan_sizes.argtypes = [_vp] + [ctypes.POINTER(i64)] * 4
    lib.sfk_plan_sizes.restype = ci
    lib.sfk_eval.argtypes = [_vp, i64, _vp, _vp, _vp, _vp, _vp]
    lib.sfk_eval.restype = ci
    lib.sfk_eval_pair.argtypes = [_vp, _vp, i64, _vp, _vp, _vp, _vp, _vp]
    lib.sfk_eval_pair.restype = ci
    lib.sfk_eval_host.argtypes = [_vp, i64, _vp, _vp, _vp, _vp, i64]
    lib.sfk_eval_host.restype = ci
    lib.sfk_sum_squares.argtypes = [_vp, i64, _vp, _vp]
    lib.sfk_sum_squares.restype = ci
    lib.sfk_launch_count.restype = i64
    lib.sfk_last_error.argtypes = [ctypes.c_char_p, i64]
    lib.sfk_last_error.restype = ci
    lib.sfk_device_info.argtypes = [ci] + [ctypes.POINTER(ci)] * 4 + [ctypes.c_char_p, ci]
    lib.sfk_device_info.restype = ci
    lib.sfk_fp64_peak.argtypes = [ctypes.c_double, _dp, _dp]
    lib.sfk_fp64_peak.restype = ci
    if hasattr(lib, "sfk_eval_gather_scatter"):   # absent from pre-(f) A/B builds
        lib.sfk_eval_gather_scatter.argtypes = [_vp, i64, _vp, _vp, _vp, _vp, _vp]
        lib.sfk_eval_gather_scatter.restype = ci
    if hasattr(lib, "sfk_eval_host_async"):
        lib.sfk_eval_host_async.argtypes = [_vp, i64, _vp, _vp, _vp, _vp, i64]
        lib.sfk_eval_host_async.restype = ci
        lib.sfk_host_wait.restype = ci
    if hasattr(lib, "sfk_eval_global"):
        lib.sfk_eval_global.argtypes = [_vp, i64, _vp, _vp, _vp, _vp, _vp, _vp]
        lib.sfk_eval_global.restype = ci
    if hasattr(lib, "sfk_csr_create"):
        lib.sfk_csr_create.argtypes = [i64, ci, _vp, i64, _vp, ctypes.POINTER(_vp)]
        lib.sfk_csr_create.restype = ci
        lib.sfk_csr_info.argtypes = [_vp, ctypes.POINTER(i64), ctypes.POINTER(i64),
                                     ctypes.POINTER(_vp), ctypes.POINTER(_vp)]
        lib.sfk_csr_info.restype = ci
        lib.sfk_csr_destroy.argtypes = [_vp]
        lib.sfk_csr_destroy.restype = ci
        lib.sfk_csr_entry_map.argtypes = [_vp, i64, ci, _vp, _vp, _vp]
        lib.sfk_csr_entry_map.restype = ci
        lib.sfk_assemble_csr.argtypes = [_vp, i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
        lib.sfk_assemble_csr.restype = ci
    if hasattr(lib, "sfk_kernel_available"):
        lib.sfk_kernel_available.argtypes = [ci] * 5
        lib.sfk_kernel_available.restype = ci
    if hasattr(lib, "sfk_set_option"):
        lib.sfk_set_option.argtypes = [ctypes.c_char_p, i64]
        lib.sfk_set_option.restype = ci
        lib.sfk_get_option.argtypes = [ctypes.c_char_p, ctypes.POINTER(i64)]
        lib.sfk_get_option.restype = ci
    if hasattr(lib, "sfk_csr_insert"):
        lib.sfk_csr_insert.argtypes = [i64, ci, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
        lib.sfk_csr_insert.restype = ci
    if hasattr(lib, "sfk_mesh_create"):
        lib.sfk_mesh_create.argtypes = [i64, ci, ctypes.POINTER(_vp)]
        lib.sfk_mesh_create.restype = ci
        lib.sfk_mesh_upload.argtypes = [_vp, _vp]
        lib.sfk_mesh_upload.restype = ci
        lib.sfk_mesh_coords.argtypes = [_vp]
        lib.sfk_mesh_coords.restype = _vp
        lib.sfk_mesh_destroy.argtypes = [_vp]
        lib.sfk_mesh_destroy.restype = ci
        lib.sfk_eval_host_mesh.argtypes = [_vp, _vp, i64, i64, _vp, _vp, _vp, i64, ci]
        lib.sfk_eval_host_mesh.restype = ci


def load_library(build_if_missing=True):
    """Load libsfk.so (building it in-tree with nvcc if it is absent)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    with _LOCK:
        if _LIB is not None:
            return _LIB
        path = library_path()
        if not os.path.exists(path):
            if not build_if_missing:
                raise NativeError(-1, "libsfk.so not built (run __graft_entry__.build())")
            from ._build import build_native
            build_native()
        lib = ctypes.CDLL(path)
        _declare(lib)
        if lib.sfk_abi_version() != ABI_VERSION:
            raise NativeError(-1, "libsfk.so ABI %d != expected %d"
                              % (lib.sfk_abi_version(), ABI_VERSION))
        _LIB = lib
        return lib


def _check(status):
    if status != 0:
        buf = ctypes.create_string_buffer(512)
        _LIB.sfk_last_error(buf, 512)
        raise NativeError(status, buf.value.decode(errors="replace"))


def _as_dp(arr):
    return arr.ctypes.data_as(_dp)


class _NativePlan:
    def __init__(self, plan):
        lib = load_library()
        h = _vp()
        params = np.asarray(plan.params, dtype=np.float64)
        _check(lib.sfk_plan_create(
            plan.kind, plan.dim, int(plan.degree), plan.n, plan.m,
            int(plan.collocated), _as_dp(plan.B), _as_dp(plan.D),
            _as_dp(plan.wq), _as_dp(plan.xq), _as_dp(plan.Bc), _as_dp(plan.Dc),
            _as_dp(params) if len(params) else None, len(params),
            ctypes.byref(h)))
        self.handle = h
        self._lib = lib

    def __del__(self):
        try:
            if self.handle:
                self._lib.sfk_plan_destroy(self.handle)
        except Exception:
            pass


def kernel_available(kind, dim, n, m, collocated):
    """The C library's instance table (sfk_kernel_available): is there a
    kernel for this (kind, cell dim, dofs/axis, points/axis, collocated)?"""
    return bool(load_library().sfk_kernel_available(int(kind), int(dim), int(n), int(m),
                                                     int(bool(collocated))))


def native_plan(plan):
    """The C-ABI plan handle of a KernelPlan (created once, cached)."""
    np_ = plan._native.get("handle")
    if np_ is None:
        np_ = _NativePlan(plan)
        plan._native["handle"] = np_
    return np_.handle


# ---------------------------------------------------------------------------
# validation (reference interpreter.py:291-299 semantics)


def _collect(plan, inputs, is_tensor):
    """Return ({name: 2D array}, ncells, squeeze) after reference checks."""
    out = {}
    ncells = None
    squeeze = False
    for name, size in plan.arguments:
        if name not in inputs:
            raise UnboundVariable(name)
        arr = inputs[name]
        shape = tuple(arr.shape)
        if len(shape) == 1:
            if shape[0] != size:
                raise ShapeMismatch("argument %s has size %d, declared %d"
                                    % (name, shape[0], size))
            arr = arr.reshape(1, size)
            squeeze = True
        elif len(shape) == 2:
            if shape[1] != size:
                raise ShapeMismatch("argument %s has per-cell size %d, declared %d"
                                    % (name, shape[1], size))
        else:
            raise ShapeMismatch("argument %s must be (ncells, %d), got %s"
                                % (name, size, shape))
        if ncells is None:
            ncells = arr.shape[0]
        elif arr.shape[0] != ncells:
            raise ShapeMismatch("argument %s has %d cells, expected %d"
                                % (name, arr.shape[0], ncells))
        out[name] = arr
    return out, (ncells or 0), squeeze


def evaluate_batched(plan, inputs, out=None, stream=None):
    """Evaluate ``plan`` on every cell of a batch.

    inputs: mapping argument name -> (ncells, size) float64 array, either
    torch CUDA tensors (stream-ordered, returns a CUDA tensor) or numpy
    arrays (synchronous host path, returns numpy).  A 1D array of one cell's
    size is accepted and a 1D result returned, like ``run_kernel``.
    """
    if getattr(plan, "meta", {}).get("backend") == "loopprogram":
        return plan.evaluate(inputs, out=out, stream=stream)
    first = next(iter(inputs.values()), None) if inputs else None
    if first is not None and isinstance(first, np.ndarray):
        return evaluate_host(plan, inputs, out=out)
    args, ncells, squeeze, dev, stream = _device_args(plan, inputs, stream)
    rsize = plan.return_size
    import torch

    if out is None:
        out = torch.empty((ncells, rsize), dtype=torch.float64, device=dev)
    else:
        _check_out(out, (ncells, rsize), dev, args)
    handle = native_plan(plan)
    with torch.cuda.device(dev):
        _check(_LIB.sfk_eval(handle, ncells, out.data_ptr(),
                             args["coords"].data_ptr(),
                             args["w0"].data_ptr() if "w0" in args else None,
                             args["w1"].data_ptr() if "w1" in args else None,
                             stream))
    return out.reshape(rsize) if squeeze else out


def evaluate_batched_pair(plan0, plan1, inputs, stream=None):
    """Two plans over the same (coords, w0) in one fused launch when the pair
    has a fused kernel (quad mass + Laplace action, BASELINE config C1).
    Same validation as ``evaluate_batched``."""
    import torch

    _collect(plan1, inputs, True)
    args, ncells, _, dev, stream = _device_args(plan0, inputs, stream)
    a0 = torch.empty((ncells, plan0.return_size), dtype=torch.float64, device=dev)
    a1 = torch.empty((ncells, plan1.return_size), dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        _check(load_library().sfk_eval_pair(
            native_plan(plan0), native_plan(plan1), ncells, a0.data_ptr(),
            a1.data_ptr(), args["coords"].data_ptr(),
            args["w0"].data_ptr() if "w0" in args else None, stream))
    return a0, a1


def _device_args(plan, inputs, stream):
    """Validate device inputs (reference interpreter.py:291-299 checks, then
    dtype / device / contiguity) and resolve the stream handle.

    Non-contiguous arguments are copied on the CURRENT torch stream; when the
    kernel runs on another ``stream`` that stream is made to wait for the
    copies and the temporaries are recorded on it, so the caching allocator
    cannot hand their memory out before the kernel has read it."""
    import torch

    args, ncells, squeeze = _collect(plan, inputs, True)
    if not torch.cuda.is_available():
        raise NativeError(-1, "evaluate_batched needs a CUDA device (no CPU fallback)")
    dev = None
    copied = []
    for name, t in args.items():
        if not isinstance(t, torch.Tensor):
            raise TypeError("argument %s must be a torch.Tensor or numpy array" % name)
        if t.dtype != torch.float64:
            raise TypeError("argument %s must be float64, got %s" % (name, t.dtype))
        if not t.is_cuda:
            raise TypeError("argument %s must live on a CUDA device" % name)
        dev = t.device if dev is None else dev
        if t.device != dev:
            raise ValueError("all arguments must be on one device")
        if not t.is_contiguous():
            args[name] = t.contiguous()
            copied.append(args[name])
    if dev is None:
        raise UnboundVariable("coords")
    cur = torch.cuda.current_stream(dev)
    if stream is None:
        stream = cur.cuda_stream
    elif copied and int(stream) != cur.cuda_stream:
        ext = torch.cuda.ExternalStream(int(stream), device=dev)
        ext.wait_stream(cur)
        for t in copied:
            t.record_stream(ext)
    return args, ncells, squeeze, dev, stream


def _check_out(out, shape, dev, args):
    import torch

    if not isinstance(out, torch.Tensor) or out.dtype != torch.float64:
        raise TypeError("out must be a float64 torch.Tensor")
    if tuple(out.shape) != shape or not out.is_contiguous():
        raise ShapeMismatch("out must be a contiguous (%d, %d) tensor" % shape)
    if out.device != dev:
        raise ValueError("out must be on %s, got %s" % (dev, out.device))
    for name, t in args.items():
        if out.numel() and t.numel() and _overlaps(out, t):
            raise ValueError("out must not alias argument %s (A is overwritten)" % name)


def _overlaps(a, b):
    a0, b0 = a.data_ptr(), b.data_ptr()
    a1 = a0 + a.numel() * a.element_size()
    b1 = b0 + b.numel() * b.element_size()
    return a0 < b1 and b0 < a1


def evaluate_host(plan, inputs, out=None, chunk_cells=0):
    """Host-buffer evaluation through ``sfk_eval_host`` (synchronous)."""
    args, ncells, squeeze = _collect(plan, inputs, False)
    for name in list(args):
        a = args[name]
        if a.dtype != np.float64:
            raise TypeError("argument %s must be float64" % name)
        if not a.flags.c_contiguous:
            args[name] = np.ascontiguousarray(a)
    rsize = plan.return_size
    if out is None:
        out = np.empty((ncells, rsize), dtype=np.float64)
    elif out.shape != (ncells, rsize) or not out.flags.c_contiguous or out.dtype != np.float64:
        raise ShapeMismatch("out must be a contiguous float64 (%d, %d) array" % (ncells, rsize))
    lib = load_library()

    def ptr(name):
        return args[name].ctypes.data if name in args else None

    _check(lib.sfk_eval_host(native_plan(plan), ncells, out.ctypes.data,
                             ptr("coords"), ptr("w0"), ptr("w1"), int(chunk_cells)))
    return out.reshape(rsize) if squeeze else out


def evaluate_host_ptrs(plan, ncells, a_ptr, coords_ptr, w0_ptr, w1_ptr, chunk_cells=0,
                       wait=True):
    """Raw-pointer host evaluation (pinned torch tensors from the bench).
    wait=False only enqueues (sfk_eval_host_async): call host_wait() before
    touching the buffers."""
    fn = load_library().sfk_eval_host if wait else load_library().sfk_eval_host_async
    _check(fn(native_plan(plan), ncells, a_ptr, coords_ptr, w0_ptr, w1_ptr, int(chunk_cells)))


def host_wait():
    """Wait for every evaluate_host_ptrs(..., wait=False) on the current device."""
    _check(load_library().sfk_host_wait())


class Mesh:
    """Device-resident cell coordinates (sfk_mesh, include/sfk.h): upload once,
    then evaluate host-side w0 / w1 -> A on any number of plans without
    re-sending the coordinates (the reference's emitted kernels take
    ``coords`` on every call, scheduling.py:731-735)."""

    def __init__(self, ncells, coords_size=24):
        import ctypes

        lib = load_library()
        h = ctypes.c_void_p()
        _check(lib.sfk_mesh_create(int(ncells), int(coords_size), ctypes.byref(h)))
        self._h, self._lib = h, lib
        self.ncells, self.coords_size = int(ncells), int(coords_size)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.sfk_mesh_destroy(h)
            self._h = None

    def upload(self, coords_ptr):
        """Asynchronous H2D of the coordinates (host pointer, ideally pinned);
        later evaluate_host calls are ordered after it."""
        _check(self._lib.sfk_mesh_upload(self._h, coords_ptr))

    def device_coords(self):
        """Device address of the [ncells][coords_size] coordinates."""
        return self._lib.sfk_mesh_coords(self._h)

    def evaluate_host_ptrs(self, plan, a_ptr, w0_ptr, w1_ptr=None, first_cell=0, ncells=None,
                           chunk_cells=0, wait=True):
        n = self.ncells - first_cell if ncells is None else ncells
        _check(self._lib.sfk_eval_host_mesh(native_plan(plan), self._h, int(first_cell), int(n),
                                            a_ptr, w0_ptr, w1_ptr, int(chunk_cells),
                                            1 if wait else 0))


def sum_squares(x, workspace=None, stream=None):
    """(sum x^2, sum x) of a CUDA float64 tensor, as a 2-element CUDA tensor
    (device-side, stream-ordered; no host sync)."""
    import torch

    if x.dtype != torch.float64 or not x.is_cuda:
        raise TypeError("sum_squares needs a CUDA float64 tensor")
    x = x.contiguous()
    if workspace is None:
        workspace = torch.empty(SUM_WORKSPACE, dtype=torch.float64, device=x.device)
    if stream is None:
        stream = torch.cuda.current_stream(x.device).cuda_stream
    with torch.cuda.device(x.device):
        _check(load_library().sfk_sum_squares(x.data_ptr(), x.numel(),
                                              workspace.data_ptr(), stream))
    return workspace[:2]


# Kernel-variant names of option "c2_kernel" (sfk_options.h OPT_C2_KERNEL).
C2_KERNELS = {"auto": 0, "v1": 1, "v2": 2, "v3": 3, "tc": 4, "cell": 5, "v4": 6, "v5": 7,
              "cellv": 8, "v6": 10, "tc8c": 11}


def set_option(name, value):
    """Set a process-wide tuning option of libsfk (A/B runs; 0 = built-in
    choice).  ``c2_kernel`` also accepts a generation name (``"v5"``)."""
    if name == "c2_kernel" and isinstance(value, str):
        value = C2_KERNELS[value]
    _check(load_library().sfk_set_option(name.encode(), int(value)))


def get_option(name):
    v = ctypes.c_int64()
    _check(load_library().sfk_get_option(name.encode(), ctypes.byref(v)))
    return v.value


@contextlib.contextmanager
def options(**values):
    """Temporarily set tuning options (restored on exit)."""
    old = {k: get_option(k) for k in values}
    try:
        for k, v in values.items():
            set_option(k, v)
        yield
    finally:
        for k, v in old.items():
            set_option(k, v)


def options_from_env(environ=None):
    """Tools only: map the round-1 ``SFK_<NAME>=value`` A/B switches onto
    set_option (the library itself reads no environment).  Returns the
    options applied."""
    env = os.environ if environ is None else environ
    applied = {}
    for key, val in env.items():
        if not key.startswith("SFK_") or key in ("SFK_LIBRARY", "SFK_NVRTC"):
            continue
        name = key[4:].lower()
        if name == "c2_kernel":
            v = C2_KERNELS[val]
        elif name in ("c2g_kernel", "c2g_small"):
            v = int(val.lstrip("v"))
        elif name in ("c5_p1", "c5_p3", "c5_p4"):
            v = 1 if val.startswith("p") else 0
        elif name in ("colloc_warps", "neo_warps", "lp_warp", "lp_fuse"):
            v = int(val) if int(val) != 0 else -1
        else:
            v = int(val)
        set_option(name, v)
        applied[name] = v
    return applied


def launch_count():
    return int(load_library().sfk_launch_count())


def fp64_peak(seconds=0.5):
    lib = load_library()
    f = ctypes.c_double()
    m = ctypes.c_double()
    _check(lib.sfk_fp64_peak(seconds, ctypes.byref(f), ctypes.byref(m)))
    return f.value, m.value


def device_info(device=0):
    lib = load_library()
    vals = [ctypes.c_int() for _ in range(4)]
    name = ctypes.create_string_buffer(256)
    _check(lib.sfk_device_info(device, *[ctypes.byref(v) for v in vals], name, 256))
    return {"sm_count": vals[0].value, "sm_clock_khz": vals[1].value,
            "mem_clock_khz": vals[2].value, "mem_bus_bits": vals[3].value,
            "name": name.value.decode()}
