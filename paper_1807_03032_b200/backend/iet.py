"""Loop-nest view (``Operator.iet``) and device plan text (``Operator.source``).

The reference exposes the IET it interprets and the C it emits
(pkg/src/stencilc/backend/operator.py:160-166, iet.py, codegen.py). The B200
backend executes clusters as device stages instead of interpreting a tree, so
``iet`` here is the loop structure *as the backend runs it*: one ``Section``
per top-level nest (hoisted per-point producers on the host, then the time
loop captured as one CUDA graph, then time-inner nests), each holding the
``Iteration`` nodes of its dimensions and one ``Stage`` per device launch
family with the statements it executes. ``source`` prints that plan with the
kernel family every statement is routed to.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import List


@dataclass
class IetNode:
    kind: str                       # Block | Section | Iteration | Stage | Expression
    name: str = ""
    children: List["IetNode"] = field(default_factory=list)
    attrs: dict = field(default_factory=dict)

    def walk(self):
        yield self
        for c in self.children:
            yield from c.walk()

    def dump(self, depth: int = 0) -> str:
        pad = "  " * depth
        extra = "".join(" %s=%s" % kv for kv in sorted(self.attrs.items()))
        line = "%s%s %s%s" % (pad, self.kind, self.name, extra)
        return "\n".join([line.rstrip()] + [c.dump(depth + 1)
                                            for c in self.children])


def _stage_kind(c) -> str:
    if c.fused is not None:
        return "fused-%s" % c.fused[0]
    if not any(d.is_time for d in c.dims):
        return "hoisted"
    if any(d.kind == "space" for d in c.dims):
        return "dense"
    mains = [e for e in c.eqs if e.lhs.func.kind != "temp"]
    if mains and all(e.is_increment for e in mains):
        return "sparse-inject"
    return "sparse-interpolate"


_KERNELS = {
    "fused-tti": "tti_g1z_tma + tti_upd1z_tma (rotated first derivatives, "
                 "both updates; csrc/tti.cu)",
    "dense": "acoustic_kernel<SO> when the program trace equals the fused "
             "op sequence (backend/fastpath.py), else the NVRTC-generated "
             "program kernel (csrc/jit.cu)",
    "sparse-inject": "sparse_inject_fast / sparse_inject_grouped "
                     "(csrc/api.cu)",
    "sparse-interpolate": "sparse_interp_fast (csrc/api.cu)",
    "hoisted": "host, numpy scalar semantics (per-point tables)",
}


def _expr_nodes(c) -> List[IetNode]:
    out = []
    for e in c.eqs:
        op = "+=" if e.is_increment else "="
        out.append(IetNode("Expression", "%r %s ..." % (e.lhs, op),
                           attrs={"temp": e.lhs.func.kind == "temp"}
                           if e.lhs.func.kind == "temp" else {}))
    return out


def build_iet(op) -> IetNode:
    from .operator import _device_phases, _time_outer
    clusters = op.clusters
    root = IetNode("Block", op.name, attrs={"mode": op.mode,
                                              "dtype": op.dtype})
    secs = iter(op.artifact.sections)
    for c in clusters:
        if any(d.is_time for d in c.dims):
            continue
        pd = [d for d in c.dims if d.kind == "sparse"]
        it = IetNode("Iteration", pd[0].name if pd else "-",
                     _expr_nodes(c), {"where": "host (once per apply)"})
        root.children.append(IetNode("Section", next(secs), [it]))
    for phase in _device_phases(clusters):
        sec = IetNode("Section", next(secs))
        if _time_outer(phase[0]):
            tloop = IetNode("Iteration", phase[0].dims[0].name,
                            attrs={"where": "device, one CUDA graph"})
            for c in phase:
                st = IetNode("Stage", _stage_kind(c),
                             attrs={"dims": ",".join(d.name for d in c.dims[1:])})
                st.children = _expr_nodes(c)
                tloop.children.append(st)
            sec.children.append(tloop)
        else:
            c = phase[0]
            st = IetNode("Stage", _stage_kind(c),
                         attrs={"dims": ",".join(d.name for d in c.dims),
                                "where": "device, t-outer sweeps"})
            st.children = _expr_nodes(c)
            sec.children.append(st)
        root.children.append(sec)
    return root


def device_source(op) -> str:
    lines = ["// operator %s: dtype=%s mode=%s (B200 device plan)"
             % (op.name, op.dtype, op.mode)]
    for sec in build_iet(op).children:
        lines.append("section %s:" % sec.name)
        for node in sec.walk():
            if node.kind == "Iteration":
                lines.append("  for %s  // %s" % (node.name,
                                                  node.attrs.get("where", "")))
            elif node.kind == "Stage":
                lines.append("    launch %s  // %s" % (
                    node.name, _KERNELS.get(node.name, "")))
    lines.append("")
    lines.append("// statements per cluster")
    for i, c in enumerate(op.clusters):
        lines.append("cluster %d [%s] dims=%s" % (
            i, _stage_kind(c), ",".join(d.name for d in c.dims)))
        for e in c.eqs:
            lines.append("  %r %s= %r" % (e.lhs, "+" if e.is_increment else "",
                                          e.rhs))
    return "\n".join(lines) + "\n"
