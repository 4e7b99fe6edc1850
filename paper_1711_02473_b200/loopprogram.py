"""Any reference kernel on the GPU: the LoopProgram path.

The reference compiles every form it knows (the registry of forms.py:246-263
on interval / quad / triangle / hex / prism cells, modes vanilla / coffee /
spectral, cli.py:211-217) into a ``LoopProgram`` (scheduling.py:87-95) and
serialises it loss-free to JSON (``scheduling.serialize_program``,
scheduling.py:465-532).  ``load_program`` takes that JSON and returns a plan
that ``evaluate_batched`` runs on the B200: libsfk parses the statement
list, generates a batched sm_100a kernel (one CTA-wide phase per loop nest,
shared-memory buffers, cells across threads; ``csrc/lp_codegen.cpp``) and
compiles it with NVRTC.  By default the generated code keeps the reference's
summation order and does not contract multiply-adds, so results are
bit-identical to the reference's emitted C compiled with
``-ffp-contract=off`` (the parity build of SURVEY.md §8(d)).

A reference user does::

    from sumfact import cli, scheduling
    text = scheduling.serialize_program(cli.compile_kernel("stokes_momentum", "hex", 2, "spectral"))

    import paper_1711_02473_b200 as sfk
    plan = sfk.load_program(text)
    A = sfk.evaluate_batched(plan, {"coords": X, "w0": ...})     # (C, return size)

The hand-written kernels of ``compile_kernel`` remain the fast path for the
BASELINE families; this path covers everything else the reference emits.
"""

from __future__ import annotations

import ctypes
import json
import os

import numpy as np

from .errors import NativeError, ShapeMismatch, UsageError
from . import runtime as _rt

__all__ = ["LoopProgramPlan", "load_program", "program_flops"]

FMA = 1
NO_JIT = 2
_CONFIG_KEYS = ("cells_per_block", "threads", "slots_per_cell", "smem_bytes",
                "global_scratch", "phases", "serial_phases", "barriers",
                "cubin_bytes", "warp_mode", "fused_phases")


def _declare(lib):
    i64 = ctypes.c_int64
    ci = ctypes.c_int
    vp = ctypes.c_void_p
    lib.sfk_program_create.argtypes = [ctypes.c_char_p, i64, ci, ctypes.POINTER(vp)]
    lib.sfk_program_create.restype = ci
    lib.sfk_program_destroy.argtypes = [vp]
    lib.sfk_program_destroy.restype = ci
    lib.sfk_program_sizes.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(ci),
                                      ctypes.POINTER(i64), ci]
    lib.sfk_program_sizes.restype = ci
    lib.sfk_program_config.argtypes = [vp, ctypes.POINTER(i64), ci]
    lib.sfk_program_config.restype = ci
    lib.sfk_program_text.argtypes = [vp, ci, ctypes.c_char_p, i64, ctypes.POINTER(i64)]
    lib.sfk_program_text.restype = ci
    lib.sfk_program_eval.argtypes = [vp, i64, vp, ctypes.POINTER(vp), ci, vp]
    lib.sfk_program_eval.restype = ci
    lib._sfk_program_declared = True


def _lib():
    lib = _rt.load_library()
    if not getattr(lib, "_sfk_program_declared", False):
        if not hasattr(lib, "sfk_program_create"):
            raise NativeError(-1, "libsfk.so predates the LoopProgram path; rebuild it")
        _declare(lib)
    return lib


def _text_of(program):
    if isinstance(program, (bytes, bytearray)):
        return bytes(program)
    if isinstance(program, dict):
        return json.dumps(program, sort_keys=True, separators=(",", ":")).encode()
    if isinstance(program, os.PathLike) or (isinstance(program, str)
                                            and not program.lstrip().startswith("{")):
        with open(program, "rb") as fh:
            return fh.read()
    if isinstance(program, str):
        return program.encode()
    raise UsageError("load_program takes the JSON text of "
                     "scheduling.serialize_program(program), a path to it, or its dict")


class LoopProgramPlan:
    """A reference LoopProgram compiled for the GPU.

    Carries the reference program's ABI metadata — ``name``,
    ``return_buffer`` ('A', size), ``arguments`` [(name, size), ...] in slot
    order (scheduling.py:87-95) — so it is accepted wherever a plan is.
    """

    def __init__(self, program, fma=False, jit=True):
        self._handle = None
        self.text = _text_of(program)
        self.fma = bool(fma)
        lib = _lib()
        h = ctypes.c_void_p()
        flags = (FMA if fma else 0) | (0 if jit else NO_JIT)
        # the native parser validates first (malformed -> NativeError / EINVAL)
        _rt._check(lib.sfk_program_create(self.text, len(self.text), flags, ctypes.byref(h)))
        self._handle = h
        self._libref = lib
        doc = json.loads(self.text)
        self.name = doc["name"]
        self.return_buffer = tuple(doc["return"])
        self.arguments = [tuple(a) for a in doc["arguments"]]
        self.temporaries = [tuple(t) for t in doc["temporaries"]]
        self.meta = {"backend": "loopprogram", "fma": self.fma}
        rs = ctypes.c_int64()
        na = ctypes.c_int()
        sizes = (ctypes.c_int64 * 8)()
        _rt._check(lib.sfk_program_sizes(h, ctypes.byref(rs), ctypes.byref(na), sizes, 8))
        if (rs.value != self.return_buffer[1]
                or [s for _, s in self.arguments] != list(sizes[:na.value])):
            raise NativeError(-1, "libsfk disagrees with the program's ABI metadata")

    def __del__(self):
        try:
            if self._handle:
                self._libref.sfk_program_destroy(self._handle)
        except Exception:
            pass

    @property
    def return_size(self):
        return int(self.return_buffer[1])

    @property
    def config(self):
        out = (ctypes.c_int64 * len(_CONFIG_KEYS))()
        _rt._check(self._libref.sfk_program_config(self._handle, out, len(_CONFIG_KEYS)))
        return dict(zip(_CONFIG_KEYS, (int(v) for v in out)))

    def _text(self, what):
        n = ctypes.c_int64()
        _rt._check(self._libref.sfk_program_text(self._handle, what, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value + 1)
        _rt._check(self._libref.sfk_program_text(self._handle, what, buf, n.value + 1, None))
        return buf.value.decode()

    @property
    def cuda_source(self):
        """The generated CUDA C++ (what NVRTC compiled)."""
        return self._text(0)

    @property
    def entry(self):
        return self._text(1)

    def evaluate(self, inputs, out=None, stream=None):
        """Device path: torch CUDA tensors in, CUDA tensor out (stream-ordered).
        numpy in -> copies through the device, numpy out (synchronous)."""
        import torch

        first = next(iter(inputs.values()), None) if inputs else None
        if first is not None and isinstance(first, np.ndarray):
            if not torch.cuda.is_available():
                raise NativeError(-1, "LoopProgram evaluation needs a CUDA device "
                                      "(no CPU fallback)")
            dev = {k: torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).cuda()
                   for k, v in inputs.items()}
            return self.evaluate(dev).cpu().numpy()
        args, ncells, squeeze = _rt._collect(self, inputs, True)
        if not torch.cuda.is_available():
            raise NativeError(-1, "LoopProgram evaluation needs a CUDA device (no CPU fallback)")
        dev = None
        for name, t in args.items():
            if not isinstance(t, torch.Tensor) or t.dtype != torch.float64 or not t.is_cuda:
                raise TypeError("argument %s must be a float64 CUDA tensor" % name)
            dev = t.device if dev is None else dev
            if t.device != dev:
                raise ValueError("all arguments must be on one device")
            if not t.is_contiguous():
                args[name] = t.contiguous()
        rsize = self.return_size
        if dev is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        if out is None:
            out = torch.empty((ncells, rsize), dtype=torch.float64, device=dev)
        elif tuple(out.shape) != (ncells, rsize) or not out.is_contiguous():
            raise ShapeMismatch("out must be a contiguous (%d, %d) tensor" % (ncells, rsize))
        ptrs = (ctypes.c_void_p * max(1, len(self.arguments)))(
            *[args[n].data_ptr() for n, _ in self.arguments])
        if stream is None:
            stream = torch.cuda.current_stream(dev).cuda_stream
        with torch.cuda.device(dev):
            _rt._check(self._libref.sfk_program_eval(self._handle, ncells, out.data_ptr(), ptrs,
                                                     len(self.arguments), stream))
        return out.reshape(rsize) if squeeze else out


_OPS = frozenset(("+", "*", "/", "pow", "min", "max", "call", "cmp"))


def _expr_ops(e):
    if not isinstance(e, list) or not e or not isinstance(e[0], str):
        return 0
    tag = e[0]
    if tag in ("lit", "indexed", "flex", "delta", "var", "table", "idx"):
        return 0
    n = 1 if tag in _OPS else 0
    return n + sum(_expr_ops(x) for x in e[1:] if isinstance(x, list))


def program_flops(program):
    """The reference's static flop count of a LoopProgram
    (``scheduling.count_flops``, scheduling.py:416-437, with the operation
    model of ``scalar_ops``, :123-131): arithmetic, function and comparison
    nodes count 1, an accumulation adds 1, loops multiply, ZeroFill, Delta and
    table loads are free.  Used as F_alg for the program path's roofline."""
    doc = json.loads(_text_of(program))

    def walk(stmts, mult):
        total = 0
        for st in stmts:
            if st[0] == "loop":
                total += walk(st[2], mult * st[1][2])
            elif st[0] == "assign":
                total += _expr_ops(st[2]) * mult
            elif st[0] == "accumulate":
                total += (_expr_ops(st[2]) + 1) * mult
        return total
    return walk(doc["body"], 1)


def load_program(program, fma=False, jit=True):
    """Compile a reference LoopProgram (its serialize_program JSON text,
    a path to it, or the parsed dict) for the GPU."""
    return LoopProgramPlan(program, fma=fma, jit=jit)
