"""Scalar kernel expressions: the per-record computational pattern.

Drop-in for the reference DSL (``simdnlp/expressions.py:34-196``).  A kernel
is a tree over ``Const`` literals, ``Field`` (a real column of the bound
table) and ``Var`` (a variable-block entry addressed by an integer column),
joined by ``Unary`` / ``Binary`` operators.  One tree is evaluated for every
record of a table; on B200 that becomes one generated fp64 device function
per distinct tree *shape* (see :mod:`.codegen`).

Two orderings defined here are load-bearing for bit-exact parity:

* :func:`walk` -- post-order DFS, lhs before rhs, shared subtrees emitted
  once (reference ``expressions.py:158-179``).  It fixes the tape order.
* :func:`var_slots` -- distinct ``(block, index column)`` pairs in first
  appearance order of that walk (reference ``expressions.py:186-196``).  It
  fixes the Jacobian/Hessian COO order.
"""

from __future__ import annotations

from typing import TYPE_CHECKING, Iterator, Union

if TYPE_CHECKING:  # pragma: no cover
    from .core import VariableBlock

UNARY_OPS = frozenset(("neg", "sin", "cos", "exp", "log", "sqrt"))
BINARY_OPS = frozenset(("add", "sub", "mul", "div", "pow"))


class Expr:
    """Base node.  Python operators build larger trees."""

    __slots__ = ()

    # binary operators: the receiver is the left operand unless reflected
    def _bin(self, op: str, other, reflected: bool = False) -> "Binary":
        o = as_expr(other)
        return Binary(op, o, self) if reflected else Binary(op, self, o)

    def __add__(self, o):
        return self._bin("add", o)

    def __radd__(self, o):
        return self._bin("add", o, True)

    def __sub__(self, o):
        return self._bin("sub", o)

    def __rsub__(self, o):
        return self._bin("sub", o, True)

    def __mul__(self, o):
        return self._bin("mul", o)

    def __rmul__(self, o):
        return self._bin("mul", o, True)

    def __truediv__(self, o):
        return self._bin("div", o)

    def __rtruediv__(self, o):
        return self._bin("div", o, True)

    def __pow__(self, o):
        return self._bin("pow", o)

    def __rpow__(self, o):
        return self._bin("pow", o, True)

    def __neg__(self):
        return Unary("neg", self)

    def __pos__(self):
        return self

    # identity semantics: a node used twice is one shared subtree
    __hash__ = object.__hash__

    def __eq__(self, other):  # noqa: D105 - identity, like the reference's eq=False
        return self is other


class Const(Expr):
    __slots__ = ("value",)

    def __init__(self, value: float):
        object.__setattr__(self, "value", float(value))

    def __setattr__(self, k, v):
        raise AttributeError("expression nodes are immutable")

    def __repr__(self) -> str:
        return f"Const({self.value!r})"


class Field(Expr):
    """A real column of the table the kernel is bound to."""

    __slots__ = ("name",)

    def __init__(self, name: str):
        object.__setattr__(self, "name", str(name))

    def __setattr__(self, k, v):
        raise AttributeError("expression nodes are immutable")

    def __repr__(self) -> str:
        return f"Field({self.name!r})"


class Var(Expr):
    """Entry of ``block`` at the flat position held by integer column ``index``."""

    __slots__ = ("block", "index")

    def __init__(self, block: "VariableBlock", index: str):
        object.__setattr__(self, "block", block)
        object.__setattr__(self, "index", index)

    def __setattr__(self, k, v):
        raise AttributeError("expression nodes are immutable")

    def __repr__(self) -> str:
        return f"Var(block={getattr(self.block, 'block_id', '?')}, index={self.index!r})"


class Unary(Expr):
    __slots__ = ("op", "child")

    def __init__(self, op: str, child: Expr):
        if op not in UNARY_OPS:
            raise ValueError(f"unknown unary op {op!r}")
        object.__setattr__(self, "op", op)
        object.__setattr__(self, "child", child)

    def __setattr__(self, k, v):
        raise AttributeError("expression nodes are immutable")

    def __repr__(self) -> str:
        return f"Unary({self.op!r}, {self.child!r})"


class Binary(Expr):
    __slots__ = ("op", "lhs", "rhs")

    def __init__(self, op: str, lhs: Expr, rhs: Expr):
        if op not in BINARY_OPS:
            raise ValueError(f"unknown binary op {op!r}")
        object.__setattr__(self, "op", op)
        object.__setattr__(self, "lhs", lhs)
        object.__setattr__(self, "rhs", rhs)

    def __setattr__(self, k, v):
        raise AttributeError("expression nodes are immutable")

    def __repr__(self) -> str:
        return f"Binary({self.op!r}, {self.lhs!r}, {self.rhs!r})"


Operand = Union[Expr, float, int]


def as_expr(value: Operand) -> Expr:
    """Promote Python numbers to ``Const``; reference ``expressions.py:125-130``."""
    if isinstance(value, Expr):
        return value
    if isinstance(value, bool):
        return Const(float(value))
    if isinstance(value, (int, float)):
        return Const(float(value))
    try:  # numpy scalars
        import numpy as _np

        if isinstance(value, _np.generic) and _np.isrealobj(value):
            return Const(float(value))
    except ImportError:  # pragma: no cover
        pass
    raise TypeError(f"cannot use {type(value).__name__} in a kernel expression")


def field(name: str) -> Field:
    return Field(name)


def sin(e: Operand) -> Expr:
    return Unary("sin", as_expr(e))


def cos(e: Operand) -> Expr:
    return Unary("cos", as_expr(e))


def exp(e: Operand) -> Expr:
    return Unary("exp", as_expr(e))


def log(e: Operand) -> Expr:
    return Unary("log", as_expr(e))


def sqrt(e: Operand) -> Expr:
    return Unary("sqrt", as_expr(e))


def _children(node: Expr) -> tuple:
    if isinstance(node, Unary):
        return (node.child,)
    if isinstance(node, Binary):
        return (node.lhs, node.rhs)
    return ()


def walk(root: Expr) -> Iterator[Expr]:
    """Children-before-parents order, lhs subtree first, each node once.

    Iterative (explicit frame stack) so deep chains cannot hit the recursion
    limit.  Equivalent ordering to reference ``expressions.py:158-179``: a
    node is marked visited when it is first *entered*, so a shared subtree is
    emitted at its first (leftmost) occurrence.
    """
    visited: set[int] = set()
    if root is None:
        return
    visited.add(id(root))
    frames: list[list] = [[root, 0]]
    while frames:
        top = frames[-1]
        kids = _children(top[0])
        advanced = False
        while top[1] < len(kids):
            kid = kids[top[1]]
            top[1] += 1
            if id(kid) not in visited:
                visited.add(id(kid))
                frames.append([kid, 0])
                advanced = True
                break
        if not advanced:
            frames.pop()
            yield top[0]


def real_fields(root: Expr) -> set[str]:
    return {n.name for n in walk(root) if isinstance(n, Field)}


def var_slots(root: Expr) -> list[tuple["VariableBlock", str]]:
    """Distinct ``(block, index column)`` pairs in first-appearance order."""
    slots: list = []
    keys: set = set()
    for node in walk(root):
        if isinstance(node, Var):
            key = (id(node.block), node.index)
            if key not in keys:
                keys.add(key)
                slots.append((node.block, node.index))
    return slots
