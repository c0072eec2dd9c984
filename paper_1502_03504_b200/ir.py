"""Stencil kernel IR: the data contract between the host API and the sm_100a kernels.

This restates the reference's kernel IR (``lopec/ir.py:33-133``) so a kernel can be
described without the reference frontend, and adds the one thing the reference
never needed: a compact, exact text serialisation that crosses the C-ABI
(``lope_kernel_compile`` in ``include/lope_b200.h``).

Semantics follow ``lopec.ir.run_body`` (``ir.py:258-308``):

* ``Const`` is a float constant; integer literals are already floats
  (``lower_kernel`` at ``ir.py:159-160``).
* ``a - b`` is ``Add(a, Neg(b))`` (``ir.py:174-175``); the builder below
  reproduces that so trees built in Python match lowered ``.lope`` kernels.
* A centre ``Read`` of an array that an earlier statement stored observes the
  pending value (``ir.py:278-280``).
* ``min``/``max`` fold left with numpy NaN semantics (``ir.py:294-297``).

Kernels can be written with the builder::

    k = KernelBuilder("heat2d", rank=2)
    u = k.array("u")
    k.store(u, u[0, 0] + 0.125 * (u[-1, 0] + u[1, 0] + u[0, -1] + u[0, 1] - 4 * u[0, 0]))
    kir = k.build()

or converted from a lowered reference kernel with :func:`from_lopec`.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Iterable, Union

MAX_HALO_WIDTH = 8          # lopec/symbols.py:25
MAX_RANK = 3                # oracle_step/lower_kernel accept rank 3
INTRINSICS = ("abs", "sqrt", "min", "max")


class _Ops:
    """Operator overloading that lowers exactly like ``lopec.ir._lower_expr``."""

    def __add__(self, o):
        return Add(self, _lift(o))

    def __radd__(self, o):
        return Add(_lift(o), self)

    def __sub__(self, o):
        return Add(self, Neg(_lift(o)))

    def __rsub__(self, o):
        return Add(_lift(o), Neg(self))

    def __mul__(self, o):
        return Mul(self, _lift(o))

    def __rmul__(self, o):
        return Mul(_lift(o), self)

    def __truediv__(self, o):
        return Div(self, _lift(o))

    def __rtruediv__(self, o):
        return Div(_lift(o), self)

    def __neg__(self):
        return Neg(self)


@dataclass(frozen=True, eq=True)
class Const(_Ops):
    value: float

    def __repr__(self):
        return f"Const({self.value!r})"


@dataclass(frozen=True, eq=True)
class ScalarRead(_Ops):
    name: str

    def __repr__(self):
        return f"ScalarRead({self.name})"


@dataclass(frozen=True, eq=True)
class Read(_Ops):
    array: str
    offsets: tuple

    def __repr__(self):
        return f"Read({self.array},{self.offsets})"


@dataclass(frozen=True, eq=True)
class Add(_Ops):
    left: object
    right: object


@dataclass(frozen=True, eq=True)
class Mul(_Ops):
    left: object
    right: object


@dataclass(frozen=True, eq=True)
class Div(_Ops):
    left: object
    right: object


@dataclass(frozen=True, eq=True)
class Neg(_Ops):
    operand: object


@dataclass(frozen=True, eq=True)
class IntrinsicCall(_Ops):
    fn: str
    args: tuple


IRExpr = Union[Const, ScalarRead, Read, Add, Mul, Div, Neg, IntrinsicCall]


def _lift(v) -> IRExpr:
    if isinstance(v, _Ops):
        return v
    if isinstance(v, bool):
        raise TypeError("booleans are not kernel values")
    if isinstance(v, (int, float)):
        return Const(float(v))
    raise TypeError(f"cannot use {type(v).__name__} in a kernel expression")


def fabs(x):
    return IntrinsicCall("abs", (_lift(x),))


def fsqrt(x):
    return IntrinsicCall("sqrt", (_lift(x),))


def fmin(*xs):
    if len(xs) < 2:
        raise ValueError("min needs at least two arguments")
    return IntrinsicCall("min", tuple(_lift(x) for x in xs))


def fmax(*xs):
    if len(xs) < 2:
        raise ValueError("max needs at least two arguments")
    return IntrinsicCall("max", tuple(_lift(x) for x in xs))


@dataclass(frozen=True)
class IRAssign:
    target: str
    is_array: bool          # True: centre store into array `target`; False: kernel-local scalar
    expr: IRExpr


@dataclass(frozen=True)
class Footprint:
    """Per-dimension (negative reach, positive reach) of a kernel's reads (checks.py:38-55)."""

    dims: tuple

    @property
    def rank(self) -> int:
        return len(self.dims)

    @staticmethod
    def zero(rank: int) -> "Footprint":
        return Footprint(tuple((0, 0) for _ in range(rank)))

    def widen(self, offsets) -> "Footprint":
        return Footprint(tuple((max(n, -o), max(p, o)) for (n, p), o in zip(self.dims, offsets)))


@dataclass
class KernelIR:
    """A lowered kernel: same fields as ``lopec.ir.KernelIR`` (ir.py:112-133)."""

    name: str
    array_params: list
    scalar_params: list
    param_rank: dict
    param_types: dict
    local_scalars: list
    footprints: dict
    body: list

    @property
    def rank(self) -> int:
        return self.param_rank[self.array_params[0]]

    @property
    def stored_arrays(self) -> list:
        seen = []
        for st in self.body:
            if st.is_array and st.target not in seen:
                seen.append(st.target)
        return seen

    def validate(self) -> None:
        """Structural checks the C side repeats; raises ValueError (E104/E101/E103 analogues)."""
        if not self.array_params:
            raise ValueError(f"kernel '{self.name}' has no array parameter")
        rank = self.rank
        if not 1 <= rank <= MAX_RANK:
            raise ValueError(f"kernel rank {rank} outside 1..{MAX_RANK}")
        for a in self.array_params:
            if self.param_rank[a] != rank:
                raise ValueError("all array parameters must share one rank")
        known_scalars = set(self.scalar_params)
        assigned = set()
        stored = set()
        for st in self.body:
            for r in _reads(st.expr):
                if r.array not in self.array_params:
                    raise ValueError(f"read of unknown array '{r.array}'")
                if len(r.offsets) != rank:
                    raise ValueError(f"read of '{r.array}' has {len(r.offsets)} offsets, rank is {rank}")
                if r.array in stored and any(o != 0 for o in r.offsets):
                    raise ValueError(f"'{r.array}' is read at a halo offset after a centre store (E103)")
                if any(abs(o) > MAX_HALO_WIDTH for o in r.offsets):
                    raise ValueError(f"offset {r.offsets} exceeds the maximum halo width {MAX_HALO_WIDTH}")
            for s in _scalar_reads(st.expr):
                if s.name not in known_scalars and s.name not in assigned:
                    raise ValueError(f"scalar '{s.name}' read before assignment")
            for c in _calls(st.expr):
                if c.fn not in INTRINSICS:
                    raise ValueError(f"intrinsic '{c.fn}' is not allowed (E104)")
            if st.is_array:
                if st.target not in self.array_params:
                    raise ValueError(f"store to unknown array '{st.target}'")
                stored.add(st.target)
            else:
                if st.target in self.array_params or st.target in self.scalar_params:
                    raise ValueError(f"cannot assign parameter '{st.target}' as a local")
                assigned.add(st.target)
        if not stored:
            raise ValueError(f"kernel '{self.name}' stores no array")


def _walk(e):
    yield e
    if isinstance(e, (Add, Mul, Div)):
        yield from _walk(e.left)
        yield from _walk(e.right)
    elif isinstance(e, Neg):
        yield from _walk(e.operand)
    elif isinstance(e, IntrinsicCall):
        for a in e.args:
            yield from _walk(a)


def _reads(e):
    return [n for n in _walk(e) if isinstance(n, Read)]


def _scalar_reads(e):
    return [n for n in _walk(e) if isinstance(n, ScalarRead)]


def _calls(e):
    return [n for n in _walk(e) if isinstance(n, IntrinsicCall)]


def compute_footprints(array_params, rank, body) -> dict:
    fps = {a: Footprint.zero(rank) for a in array_params}
    for st in body:
        for r in _reads(st.expr):
            fps[r.array] = fps[r.array].widen(r.offsets)
    return fps


# ---------------------------------------------------------------------------
# Builder


class ArrayParam:
    def __init__(self, name: str, rank: int):
        self.name = name
        self.rank = rank

    def __getitem__(self, offsets):
        if not isinstance(offsets, tuple):
            offsets = (offsets,)
        if len(offsets) != self.rank:
            raise ValueError(f"'{self.name}' has rank {self.rank}, got {len(offsets)} offsets")
        if not all(isinstance(o, int) and not isinstance(o, bool) for o in offsets):
            raise TypeError("offsets must be integer literals")
        return Read(self.name, tuple(int(o) for o in offsets))


class KernelBuilder:
    """Build a ``KernelIR`` in Python: the local-element kernel definition of the API."""

    def __init__(self, name: str, rank: int):
        if not 1 <= rank <= MAX_RANK:
            raise ValueError(f"rank {rank} outside 1..{MAX_RANK}")
        self.name = name
        self.rank = rank
        self._arrays: list = []
        self._scalars: list = []
        self._types: dict = {}
        self._locals: list = []
        self._body: list = []

    def array(self, name: str) -> ArrayParam:
        name = name.lower()
        self._arrays.append(name)
        self._types[name] = "real"
        return ArrayParam(name, self.rank)

    def scalar(self, name: str, kind: str = "real") -> ScalarRead:
        if kind not in ("real", "integer"):
            raise ValueError("scalar kind must be 'real' or 'integer'")
        name = name.lower()
        self._scalars.append(name)
        self._types[name] = kind
        return ScalarRead(name)

    def let(self, name: str, expr) -> ScalarRead:
        name = name.lower()
        if name not in self._locals:
            self._locals.append(name)
            self._types[name] = "real"
        self._body.append(IRAssign(name, False, _lift(expr)))
        return ScalarRead(name)

    def store(self, arr: ArrayParam, expr) -> None:
        self._body.append(IRAssign(arr.name, True, _lift(expr)))

    def build(self) -> KernelIR:
        kir = KernelIR(self.name, list(self._arrays), list(self._scalars),
                       {a: self.rank for a in self._arrays}, dict(self._types),
                       list(self._locals),
                       compute_footprints(self._arrays, self.rank, self._body),
                       list(self._body))
        kir.validate()
        return kir


# ---------------------------------------------------------------------------
# Conversion from the reference's lowered IR (duck-typed: no import of lopec)


def from_lopec(kir) -> KernelIR:
    """Convert a ``lopec.ir.KernelIR`` (ir.py:112) into this package's IR."""

    def conv(e):
        cls = type(e).__name__
        if cls == "Const":
            return Const(float(e.value))
        if cls == "ScalarRead":
            return ScalarRead(e.name)
        if cls == "Read":
            return Read(e.array, tuple(int(o) for o in e.offsets))
        if cls == "Add":
            return Add(conv(e.left), conv(e.right))
        if cls == "Mul":
            return Mul(conv(e.left), conv(e.right))
        if cls == "Div":
            return Div(conv(e.left), conv(e.right))
        if cls == "Neg":
            return Neg(conv(e.operand))
        if cls == "IntrinsicCall":
            return IntrinsicCall(e.fn, tuple(conv(a) for a in e.args))
        raise TypeError(f"unknown IR node {cls}")

    body = [IRAssign(st.target, bool(st.is_array), conv(st.expr)) for st in kir.body]
    rank = kir.param_rank[kir.array_params[0]]
    out = KernelIR(kir.name, list(kir.array_params), list(kir.scalar_params),
                   dict(kir.param_rank), dict(kir.param_types), list(kir.local_scalars),
                   compute_footprints(list(kir.array_params), rank, body), body)
    out.validate()
    return out


# ---------------------------------------------------------------------------
# Text serialisation (the bytes that cross lope_kernel_compile)
#
#   LOPE1
#   kernel <name> <rank>
#   array <name>                   (one per array parameter, in order)
#   scalar <name> real|integer     (one per scalar parameter, in order)
#   local <name>
#   store <array> <expr>           (centre store)
#   let <local> <expr>
#   end
#
# <expr> is prefix notation: c <hexfloat> | s <name> | r <array> <o1>..<orank>
#   | + e e | * e e | / e e | n e | abs e | sqrt e | min <k> e.. | max <k> e..
# Constants are C99 hex floats, so values cross the boundary exactly.


def _ser(e, out: list) -> None:
    if isinstance(e, Const):
        out += ["c", float(e.value).hex()]
    elif isinstance(e, ScalarRead):
        out += ["s", e.name]
    elif isinstance(e, Read):
        out += ["r", e.array] + [str(int(o)) for o in e.offsets]
    elif isinstance(e, Add):
        out.append("+"); _ser(e.left, out); _ser(e.right, out)
    elif isinstance(e, Mul):
        out.append("*"); _ser(e.left, out); _ser(e.right, out)
    elif isinstance(e, Div):
        out.append("/"); _ser(e.left, out); _ser(e.right, out)
    elif isinstance(e, Neg):
        out.append("n"); _ser(e.operand, out)
    elif isinstance(e, IntrinsicCall):
        if e.fn in ("abs", "sqrt"):
            if len(e.args) != 1:
                raise ValueError(f"{e.fn} takes one argument")
            out.append(e.fn); _ser(e.args[0], out)
        elif e.fn in ("min", "max"):
            out += [e.fn, str(len(e.args))]
            for a in e.args:
                _ser(a, out)
        else:
            raise ValueError(f"unknown intrinsic {e.fn}")
    else:
        raise TypeError(f"cannot serialise {type(e).__name__}")


def serialize(kir: KernelIR) -> str:
    kir.validate()
    lines = ["LOPE1", f"kernel {kir.name} {kir.rank}"]
    lines += [f"array {a}" for a in kir.array_params]
    lines += [f"scalar {s} {kir.param_types.get(s, 'real')}" for s in kir.scalar_params]
    lines += [f"local {s}" for s in kir.local_scalars]
    for st in kir.body:
        toks: list = []
        _ser(st.expr, toks)
        lines.append(("store " if st.is_array else "let ") + st.target + " " + " ".join(toks))
    lines.append("end")
    return "\n".join(lines) + "\n"


def deserialize(text: str) -> KernelIR:
    lines = [ln for ln in text.splitlines() if ln.strip()]
    if not lines or lines[0].strip() != "LOPE1":
        raise ValueError("not a LOPE1 kernel")
    name, rank = None, None
    arrays, scalars, types, locs, body = [], [], {}, [], []
    for ln in lines[1:]:
        t = ln.split()
        if t[0] == "kernel":
            name, rank = t[1], int(t[2])
        elif t[0] == "array":
            arrays.append(t[1]); types[t[1]] = "real"
        elif t[0] == "scalar":
            scalars.append(t[1]); types[t[1]] = t[2]
        elif t[0] == "local":
            locs.append(t[1]); types[t[1]] = "real"
        elif t[0] in ("store", "let"):
            pos = [2]

            def parse():
                tok = t[pos[0]]; pos[0] += 1
                if tok == "c":
                    v = float.fromhex(t[pos[0]]); pos[0] += 1
                    return Const(v)
                if tok == "s":
                    v = t[pos[0]]; pos[0] += 1
                    return ScalarRead(v)
                if tok == "r":
                    a = t[pos[0]]
                    offs = tuple(int(x) for x in t[pos[0] + 1: pos[0] + 1 + rank])
                    pos[0] += 1 + rank
                    return Read(a, offs)
                if tok in "+*/":
                    l_ = parse(); r_ = parse()
                    return {"+": Add, "*": Mul, "/": Div}[tok](l_, r_)
                if tok == "n":
                    return Neg(parse())
                if tok in ("abs", "sqrt"):
                    return IntrinsicCall(tok, (parse(),))
                if tok in ("min", "max"):
                    k = int(t[pos[0]]); pos[0] += 1
                    return IntrinsicCall(tok, tuple(parse() for _ in range(k)))
                raise ValueError(f"bad token {tok!r}")

            body.append(IRAssign(t[1], t[0] == "store", parse()))
        elif t[0] == "end":
            break
        else:
            raise ValueError(f"bad line {ln!r}")
    kir = KernelIR(name, arrays, scalars, {a: rank for a in arrays}, types, locs,
                   compute_footprints(arrays, rank, body), body)
    kir.validate()
    return kir


def reads_of(kir: KernelIR) -> list:
    """Every Read node in statement order (used by the host to pick a kernel template)."""
    out = []
    for st in kir.body:
        out.extend(_reads(st.expr))
    return out


def count_flops(kir: KernelIR) -> int:
    """Arithmetic ops per point (Add/Mul/Div/Neg/intrinsics), for reporting only."""
    n = 0
    for st in kir.body:
        for node in _walk(st.expr):
            if isinstance(node, (Add, Mul, Div, Neg)):
                n += 1
            elif isinstance(node, IntrinsicCall):
                n += max(1, len(node.args) - 1)
    return n
