"""CPU oracle of the LoopProgram path — TEST INFRASTRUCTURE ONLY (see
oracle/__init__.py).

A restatement of the reference's literal program executor
``interpreter.run_kernel`` (reference interpreter.py:279-378) over the
loss-free JSON form of a LoopProgram (scheduling.py:465-596), vectorised
across cells: every buffer element is a numpy vector over the batch, loops
run in Python in program order, so each cell sees exactly the reference's
operation sequence (IEEE fp64 +, -, *, /, fabs; no contraction) and results
are bit-identical to the reference's emitted C built with -ffp-contract=off.

    run_program(json_text, {"coords": (C, 24), "w0": (C, n)}) -> (C, return size)
"""

from __future__ import annotations

import json
import math

import numpy as np

_FUNCS = {"sqrt": np.sqrt, "sin": np.sin, "cos": np.cos, "tan": np.tan,
          "exp": np.exp, "ln": np.log, "abs": np.abs}
_CMPS = {"<": np.less, ">": np.greater, "<=": np.less_equal,
         ">=": np.greater_equal, "==": np.equal, "!=": np.not_equal}


def _row_major(shape):
    s, acc = [], 1
    for e in reversed(shape):
        s.append(acc)
        acc *= e
    return tuple(reversed(s))


class _Compiler:
    """JSON expression / statement -> Python closures over (env, bufs)."""

    def __init__(self):
        self.nidx = 0

    def entry(self, e):
        if isinstance(e, list):
            self.nidx = max(self.nidx, e[1] + 1)
            k = e[1]
            return lambda env, k=k: env[k]
        v = int(e)
        return lambda env, v=v: v

    def address(self, offset, terms):
        parts = []
        const = int(offset)
        for ent, stride in terms:
            if isinstance(ent, list):
                self.nidx = max(self.nidx, ent[1] + 1)
                parts.append((ent[1], int(stride)))
            else:
                const += int(ent) * int(stride)
        if not parts:
            return lambda env, c=const: c
        if len(parts) == 1:
            (k, s), = parts
            return lambda env, c=const, k=k, s=s: c + s * env[k]
        return lambda env, c=const, p=tuple(parts): c + sum(s * env[k] for k, s in p)

    def expr(self, e):
        tag = e[0]
        if tag == "lit":
            v = float(e[1])
            return lambda env, b, v=v: v
        if tag == "indexed":
            base, mi = e[1], e[2]
            if base[0] == "table":
                shape = base[1]
                arr = np.array(base[2], dtype=np.float64)
                addr = self.address(0, list(zip(mi, _row_major(shape))))
                vals = [float(x) for x in arr]
                return lambda env, b, a=addr, t=vals: t[a(env)]
            if base[0] == "var":
                name = base[1]
                addr = self.address(0, list(zip(mi, _row_major(base[2]))))
                return lambda env, b, a=addr, n=name: b[n][a(env)]
            raise ValueError("indexed base %r" % base[0])
        if tag == "flex":
            name = e[1][1]
            addr = self.address(e[2], e[3])
            return lambda env, b, a=addr, n=name: b[n][a(env)]
        if tag == "delta":
            i, j = self.entry(e[1]), self.entry(e[2])
            return lambda env, b, i=i, j=j: 1.0 if i(env) == j(env) else 0.0
        if tag in ("+", "*", "/", "pow", "min", "max"):
            x, y = self.expr(e[1]), self.expr(e[2])
            if tag == "+":
                return lambda env, b, x=x, y=y: x(env, b) + y(env, b)
            if tag == "*":
                return lambda env, b, x=x, y=y: x(env, b) * y(env, b)
            if tag == "/":
                return lambda env, b, x=x, y=y: x(env, b) / y(env, b)
            if tag == "pow":
                return lambda env, b, x=x, y=y: np.power(x(env, b), y(env, b))
            if tag == "min":
                return lambda env, b, x=x, y=y: np.fmin(x(env, b), y(env, b))
            return lambda env, b, x=x, y=y: np.fmax(x(env, b), y(env, b))
        if tag == "call":
            f = _FUNCS[e[1]]
            x = self.expr(e[2])
            return lambda env, b, f=f, x=x: f(x(env, b))
        if tag == "cmp":
            f = _CMPS[e[1]]
            x, y = self.expr(e[2]), self.expr(e[3])
            return lambda env, b, f=f, x=x, y=y: np.where(f(x(env, b), y(env, b)), 1.0, 0.0)
        raise ValueError("cannot interpret %r" % tag)

    def stmt(self, st):
        tag = st[0]
        if tag == "loop":
            k, ext = st[1][1], st[1][2]
            self.nidx = max(self.nidx, k + 1)
            body = [self.stmt(s) for s in st[2]]

            def run(env, b, k=k, ext=ext, body=body):
                for v in range(ext):
                    env[k] = v
                    for s in body:
                        s(env, b)
            return run
        if tag in ("assign", "accumulate"):
            name, off, terms = st[1]
            addr = self.address(off, terms)
            x = self.expr(st[2])
            if tag == "assign":
                def run(env, b, n=name, a=addr, x=x):
                    b[n][a(env)] = x(env, b)
            else:
                def run(env, b, n=name, a=addr, x=x):
                    i = a(env)
                    b[n][i] = b[n][i] + x(env, b)
            return run
        if tag == "zero":
            name = st[1]

            def run(env, b, n=name):
                b[n][:] = 0.0
            return run
        raise ValueError("unknown statement %r" % tag)


def run_program(program, inputs):
    """Execute the serialized LoopProgram on a batch of cells (numpy, fp64)."""
    doc = json.loads(program) if isinstance(program, (str, bytes, bytearray)) else program
    comp = _Compiler()
    body = [comp.stmt(s) for s in doc["body"]]
    rname, rsize = doc["return"]
    ncells = None
    bufs = {}
    for name, size in doc["arguments"]:
        arr = np.asarray(inputs[name], dtype=np.float64).reshape(-1, size)
        ncells = arr.shape[0] if ncells is None else ncells
        assert arr.shape[0] == ncells
        bufs[name] = [arr[:, k].copy() for k in range(size)]   # element -> (C,) vector
    ncells = ncells or 0
    zeros = lambda n: np.zeros((n, ncells))  # noqa: E731
    bufs[rname] = zeros(rsize)
    for name, size in doc["temporaries"]:
        bufs[name] = zeros(size)
    for name in list(bufs):
        if isinstance(bufs[name], list):
            bufs[name] = np.array(bufs[name]) if bufs[name] else zeros(0)
    env = [0] * max(1, comp.nidx)
    for s in body:
        s(env, bufs)
    return np.ascontiguousarray(bufs[rname].T)


def program_iterations(program):
    """Innermost statement executions per cell (cost estimate for tests)."""
    doc = json.loads(program) if isinstance(program, (str, bytes, bytearray)) else program

    def count(stmts):
        n = 0
        for st in stmts:
            if st[0] == "loop":
                n += st[1][2] * count(st[2])
            else:
                n += 1
        return n
    return count(doc["body"])


__all__ = ["run_program", "program_iterations", "math"]
