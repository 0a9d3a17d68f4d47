"""Random scope programs for the P1 lowering / runtime tests.

A scope program is, per stream role (warp group), a list of ops:
("start", label), ("end", label), ("loop", trips), ("endloop",) -- the
record and loop instructions of a reference KernelProgram (ir.hpp).  to_kir
renders one as the reference's text IR so the same program can be lowered and
simulated by the reference (oracle/_ref ref_lower_kir).
"""
from __future__ import annotations

import json
import random

LABELS = ["A", "B", "C", "Load K", "Load K.wait", "mma", "mma.wait", "epi"]


def valid_body(rng: random.Random, depth_budget: int = 4, max_ops: int = 14):
    """A properly nested body: scopes and loops, every scope closed in the
    loop scope it opened in."""
    out = []

    def block(depth, budget):
        n = rng.randint(1, 3)
        for _ in range(n):
            if budget[0] <= 0:
                return
            r = rng.random()
            if r < 0.25 and depth < depth_budget:
                out.append(("loop", rng.randint(1, 4)))
                budget[0] -= 1
                block(depth + 1, budget)
                out.append(("endloop",))
            else:
                lab = rng.choice(LABELS)
                out.append(("start", lab))
                budget[0] -= 1
                if rng.random() < 0.5 and depth < depth_budget:
                    block(depth + 1, budget)
                out.append(("end", lab))

    block(0, [max_ops])
    return out


def mutate(rng: random.Random, body):
    """One pairing violation: a swapped end label, an end moved across a loop
    boundary, a dropped end, or a stray end."""
    body = list(body)
    kinds = ["relabel", "drop_end", "stray_end", "cross"]
    k = rng.choice(kinds)
    ends = [i for i, o in enumerate(body) if o[0] == "end"]
    if k == "relabel" and ends:
        i = rng.choice(ends)
        body[i] = ("end", rng.choice([l for l in LABELS if l != body[i][1]]))
    elif k == "drop_end" and ends:
        del body[rng.choice(ends)]
    elif k == "cross":
        # a scope that opens outside a loop and closes inside it (or the
        # reverse)
        lab = rng.choice(LABELS)
        if rng.random() < 0.5:
            body = [("start", lab), ("loop", 2), ("end", lab), ("endloop",)] + body
        else:
            body = [("loop", 2), ("start", lab), ("endloop",), ("end", lab)] + body
    else:
        body.insert(rng.randint(0, len(body)), ("end", rng.choice(LABELS)))
    return body


def to_kir(bodies, smem: int, name: str = "prog") -> str:
    lines = [f"kernel {name} wgs={len(bodies)} smem={smem} {{"]
    for k, body in enumerate(bodies):
        lines.append(f"  wg{k} {{")
        ind = 4
        for o in body:
            if o[0] == "loop":
                lines.append(" " * ind + f"for {o[1]} {{")
                ind += 2
            elif o[0] == "endloop":
                ind -= 2
                lines.append(" " * ind + "}")
            else:
                lines.append(" " * ind + f"record {o[0]} {json.dumps(o[1])}")
        lines.append("  }")
    lines.append("}")
    return "\n".join(lines) + "\n"


def dynamic_records(body) -> int:
    count, scale = 0, [1]
    for o in body:
        if o[0] == "loop":
            scale.append(scale[-1] * o[1])
        elif o[0] == "endloop":
            scale.pop()
        else:
            count += scale[-1]
    return count
