"""Kernel tapes and pattern keys.

A tape is the kernel tree flattened into instructions in :func:`walk` order
(reference ``autodiff.py:77-122``).  Instruction tuples use the reference's
vocabulary so the two can be compared directly in tests:

``("const", value)``, ``("field", name)``, ``("var", slot)``,
``(unary_op, child)``, ``(binary_op, lhs, rhs)``, ``("ipow", base, n)``.

``pow`` with a constant integral exponent becomes ``ipow`` (reference
``autodiff.py:117-118``); the exponent is then structural.

The *pattern key* is the tape with field names replaced by their
first-appearance ordinal, plus the slot -> (block class, index column)
structure.  Terms sharing a key share one generated device function; the
per-term data (field columns, index columns, block offsets) is passed at run
time.  Constant values stay in the key: they are emitted as exact hex-float
literals so that structural-zero folding (reference ``_is_zero``,
``autodiff.py:69-70``) is decided at generation time exactly as the
reference decides it at run time.
"""

from __future__ import annotations

from .expressions import Binary, Const, Expr, Field, Unary, Var, var_slots, walk


class TermTape:
    """Flattened kernel: instructions plus the ordered variable slots."""

    __slots__ = ("kernel", "slots", "k", "instr", "root", "field_names", "index_names")

    def __init__(self, kernel: Expr):
        self.kernel = kernel
        self.slots = var_slots(kernel)
        self.k = len(self.slots)
        slot_of = {(id(b), ix): s for s, (b, ix) in enumerate(self.slots)}
        position: dict[int, int] = {}
        instr: list[tuple] = []
        fields: list[str] = []
        for node in walk(kernel):
            position[id(node)] = len(instr)
            if isinstance(node, Const):
                instr.append(("const", node.value))
            elif isinstance(node, Field):
                instr.append(("field", node.name))
                if node.name not in fields:
                    fields.append(node.name)
            elif isinstance(node, Var):
                instr.append(("var", slot_of[(id(node.block), node.index)]))
            elif isinstance(node, Unary):
                instr.append((node.op, position[id(node.child)]))
            elif isinstance(node, Binary):
                lhs, rhs = position[id(node.lhs)], position[id(node.rhs)]
                if (
                    node.op == "pow"
                    and isinstance(node.rhs, Const)
                    and float(node.rhs.value).is_integer()
                ):
                    instr.append(("ipow", lhs, int(node.rhs.value)))
                else:
                    instr.append((node.op, lhs, rhs))
            else:  # pragma: no cover - the DSL has no other node kinds
                raise TypeError(f"unknown node {node!r}")
        self.instr = instr
        self.root = len(instr) - 1
        self.field_names = fields
        # distinct index columns in slot order
        idx: list[str] = []
        for _, ix in self.slots:
            if ix not in idx:
                idx.append(ix)
        self.index_names = idx

    def pattern_key(self) -> tuple:
        """Shape of the kernel, independent of column names and block offsets.

        Includes which slots share an index column and which share a
        variable block: both change the generated code (one load per index
        column; duplicate-variable doubling is only possible within a block,
        reference ``autodiff.py:492-497``).
        """
        fpos = {n: i for i, n in enumerate(self.field_names)}
        ipos = {n: i for i, n in enumerate(self.index_names)}
        norm = []
        for ins in self.instr:
            if ins[0] == "field":
                norm.append(("field", fpos[ins[1]]))
            elif ins[0] == "const":
                # repr of float is exact (shortest round-trip)
                norm.append(("const", float(ins[1]).hex()))
            else:
                norm.append(ins)
        blocks: list[int] = []
        block_class: list[int] = []
        for b, _ in self.slots:
            if id(b) not in blocks:
                blocks.append(id(b))
            block_class.append(blocks.index(id(b)))
        slot_struct = tuple(
            (block_class[s], ipos[ix]) for s, (_, ix) in enumerate(self.slots)
        )
        return (tuple(norm), slot_struct, len(self.field_names), len(self.index_names))
