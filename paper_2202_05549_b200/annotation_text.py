"""Light textual view of an annotation: (argument, mode) per access, in order.

Only used to derive the signature of synthesized gather kernels; the real parser (with
positions, linear expressions and errors) is the native one behind mt_launch.
"""
from __future__ import annotations

import re

_ACCESS = re.compile(r"^\s*(read|write|readwrite|reduce\s*\([^)]*\))\s+([A-Za-z_][A-Za-z0-9_]*)\s*\[")


def accesses(text: str) -> list[tuple[str, str]]:
    if "=>" not in text:
        return []
    body = text.split("=>", 1)[1]
    parts, depth, cur = [], 0, ""
    for ch in body:
        if ch == "[":
            depth += 1
        elif ch == "]":
            depth -= 1
        if ch == "," and depth == 0:
            parts.append(cur)
            cur = ""
        else:
            cur += ch
    if cur.strip():
        parts.append(cur)
    out = []
    for p in parts:
        m = _ACCESS.match(p)
        if not m:
            continue
        mode = "reduce" if m.group(1).startswith("reduce") else m.group(1)
        out.append((m.group(2), mode))
    return out
