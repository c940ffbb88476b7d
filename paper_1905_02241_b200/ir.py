"""Serialisable mechanism IR: the lowered `MechanismLayout` as plain data.

The reference compiler's front-end (parse -> passes -> solver lowering ->
`build_layout`, /root/reference/pkg/src/modlc/pipeline.py:35-59) produces a
`MechanismLayout` (modlc/layout.py:53-77) whose kernels are trees of
`modlc.ast_nodes.Node` (modlc/ast_nodes.py:101-137).  The CUDA backend consumes
exactly that object.  `MechIR` is a structural mirror of it that

* is built from a live `MechanismLayout` by duck typing (`from_layout`), so
  the reference front-end stays the user-facing compiler, and
* round-trips through JSON (`to_json` / `from_json`), so a GPU box that has no
  copy of the reference front-end can still print, build and run kernels for
  mechanisms compiled elsewhere (fixtures under ``fixtures/ir``).

Field meanings are the reference's; see the citations on each class.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import Any, Iterator

BUILTIN_FUNCTIONS = ("exp", "log", "pow", "sqrt", "fabs")  # modlc/symtab.py:17
KERNEL_ORDER = ("initialize", "state_update", "current_update")  # modlc/codegen.py:21
CONDUCTANCE_PERTURBATION = 0.001  # modlc/odes.py:45
NEWTON_TOL = 1e-12  # modlc/odes.py:41
NEWTON_MAX_ITER = 50  # modlc/odes.py:42

_TUPLE_ATTRS = ("names", "unknowns", "states", "solve_targets")


class Node:
    """Lowered AST node: kind tag, ordered children, attribute payload.

    Mirrors `modlc.ast_nodes.Node` (modlc/ast_nodes.py:101-137) minus spans
    and scopes, which no kernel semantics depend on.
    """

    __slots__ = ("kind", "children", "attrs")

    def __init__(self, kind: str, children=(), attrs: dict | None = None):
        self.kind = kind
        self.children = tuple(children)
        self.attrs = dict(attrs or {})

    def __repr__(self) -> str:
        tag = self.attrs.get("name") or self.attrs.get("op") or self.attrs.get("value", "")
        return f"<{self.kind} {tag} ({len(self.children)})>"

    def to_obj(self) -> dict:
        out: dict[str, Any] = {"k": self.kind}
        if self.children:
            out["c"] = [c.to_obj() for c in self.children]
        attrs = {}
        for key, val in self.attrs.items():
            if val is None:
                continue
            attrs[key] = list(val) if isinstance(val, tuple) else val
        if attrs:
            out["a"] = attrs
        return out

    @classmethod
    def from_obj(cls, obj: dict) -> "Node":
        attrs = dict(obj.get("a", {}))
        for key in _TUPLE_ATTRS:
            if key in attrs:
                attrs[key] = tuple(
                    tuple(x) if isinstance(x, list) else x for x in attrs[key]
                )
        if obj["k"] == "Number":
            attrs["value"] = float(attrs["value"])
        return cls(obj["k"], [cls.from_obj(c) for c in obj.get("c", [])], attrs)


def iter_nodes(node: Node) -> Iterator[Node]:
    """Pre-order traversal (modlc/ast_nodes.py:174-180)."""
    yield node
    for child in node.children:
        yield from iter_nodes(child)


@dataclass(frozen=True)
class Slot:
    """One dense per-instance SoA array (modlc/layout.py:38-44)."""

    name: str
    role: str  # parameter | assigned | state | ion
    index: int
    default: float | None = None
    ion_kind: str | None = None  # reversal | current | conc | None


@dataclass
class MechIR:
    """Mirror of `MechanismLayout` (modlc/layout.py:53-77)."""

    mechanism: str
    slots: list[Slot]
    global_scalars: dict[str, float]
    kernels: dict[str, tuple[Node, ...]]
    functions: dict[str, Node]
    currents: list[tuple[str, str]]
    conductance_hints: dict[str, str]
    point_process: bool = False
    verbatim_blocks: tuple[str, ...] = ()
    source: str = ""  # provenance note (file name, passes)
    meta: dict = field(default_factory=dict)

    # -- reference-compatible accessors --------------------------------
    def slot_names(self) -> list[str]:
        return [s.name for s in self.slots]

    def slot(self, name: str) -> Slot | None:
        for s in self.slots:
            if s.name == name:
                return s
        return None

    @property
    def analytic_conductance(self) -> bool:
        """modlc/layout.py:74-77."""
        return all(var in self.conductance_hints for var, _ in self.currents)

    # -- serialisation ---------------------------------------------------
    def to_obj(self) -> dict:
        return {
            "format": "nmodl-b200-ir/1",
            "mechanism": self.mechanism,
            "source": self.source,
            "meta": self.meta,
            "slots": [
                [s.name, s.role, s.index, s.default, s.ion_kind] for s in self.slots
            ],
            "global_scalars": [[k, v] for k, v in self.global_scalars.items()],
            "kernels": {k: [s.to_obj() for s in v] for k, v in self.kernels.items()},
            "functions": {k: v.to_obj() for k, v in self.functions.items()},
            "currents": [list(c) for c in self.currents],
            "conductance_hints": self.conductance_hints,
            "point_process": self.point_process,
            "verbatim_blocks": list(self.verbatim_blocks),
        }

    def to_json(self) -> str:
        return json.dumps(self.to_obj(), indent=1, sort_keys=False) + "\n"

    @classmethod
    def from_obj(cls, obj: dict) -> "MechIR":
        if obj.get("format") != "nmodl-b200-ir/1":
            raise ValueError("not an nmodl-b200 IR document")
        return cls(
            mechanism=obj["mechanism"],
            slots=[Slot(n, r, i, d, k) for n, r, i, d, k in obj["slots"]],
            global_scalars={k: float(v) for k, v in obj["global_scalars"]},
            kernels={k: tuple(Node.from_obj(s) for s in v) for k, v in obj["kernels"].items()},
            functions={k: Node.from_obj(v) for k, v in obj["functions"].items()},
            currents=[(a, b) for a, b in obj["currents"]],
            conductance_hints=dict(obj["conductance_hints"]),
            point_process=bool(obj["point_process"]),
            verbatim_blocks=tuple(obj["verbatim_blocks"]),
            source=obj.get("source", ""),
            meta=obj.get("meta", {}),
        )

    @classmethod
    def from_json(cls, text: str) -> "MechIR":
        return cls.from_obj(json.loads(text))

    @classmethod
    def load(cls, path) -> "MechIR":
        with open(path, "r", encoding="utf-8") as fh:
            return cls.from_json(fh.read())


def _convert_node(node) -> Node:
    return Node(node.kind, [_convert_node(c) for c in node.children], dict(node.attrs))


def from_layout(layout, source: str = "") -> MechIR:
    """Convert a reference `MechanismLayout` (duck-typed) into `MechIR`.

    Accepts a `MechIR` unchanged, so every public entry point of this package
    takes either form.
    """
    if isinstance(layout, MechIR):
        return layout
    kernels = {}
    for name, kernel in layout.kernels.items():
        kernels[name] = tuple(_convert_node(s) for s in kernel.statements)
    return MechIR(
        mechanism=layout.mechanism,
        slots=[Slot(s.name, s.role, s.index, s.default, s.ion_kind) for s in layout.slots],
        global_scalars=dict(layout.global_scalars),
        kernels=kernels,
        functions={k: _convert_node(v) for k, v in layout.functions.items()},
        currents=[tuple(c) for c in layout.currents],
        conductance_hints=dict(layout.conductance_hints),
        point_process=bool(layout.point_process),
        verbatim_blocks=tuple(layout.verbatim_blocks),
        source=source,
    )


def newton_parts(node: Node):
    """Residual and Jacobian children of a NewtonSolveNode (modlc/odes.py:545-551)."""
    n = node.attrs["n"]
    residuals = list(node.children[:n])
    flat = node.children[n : n + n * n]
    return residuals, [list(flat[i * n : (i + 1) * n]) for i in range(n)]


def linear_parts(node: Node):
    """Matrix and RHS children of a LinearSolveNode (modlc/odes.py:554-560)."""
    n = node.attrs["n"]
    flat = node.children[: n * n]
    return [list(flat[i * n : (i + 1) * n]) for i in range(n)], list(node.children[n * n : n * n + n])


def mangle(name: str) -> str:
    """C identifier for an (indexed) slot name (modlc/codegen.py:31-32)."""
    return name.replace("[", "_").replace("]", "")
