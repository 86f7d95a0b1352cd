"""Byte-stable JSON writer shared by profiles, plans, traces and reports.

Contract (reference serialize.py:1-63): one line, ``", "`` / ``": "``
separators, floats printed with 17 significant digits (``%.17g`` round-trips
every binary64), booleans/null in JSON spelling, a trailing newline.  Profile
documents sort their keys; plan documents keep insertion order.
"""

from __future__ import annotations

import math
from typing import Any

__all__ = ["format_float", "dumps_canonical"]


def format_float(value: float) -> str:
    """17-significant-digit rendering; refuses NaN/inf (not valid JSON)."""
    if math.isnan(value) or math.isinf(value):
        raise ValueError(f"cannot serialize non-finite float {value!r}")
    return "%.17g" % value


def _quote(text: str) -> str:
    return '"' + text.replace("\\", "\\\\").replace('"', '\\"') + '"'


def _render(node: Any, sort_keys: bool, sink: list) -> None:
    # bool must be tested before int (bool is an int subclass)
    if node is None:
        sink.append("null")
        return
    if node is True or node is False:
        sink.append("true" if node else "false")
        return
    if isinstance(node, int):
        sink.append(str(node))
        return
    if isinstance(node, float):
        sink.append(format_float(node))
        return
    if isinstance(node, str):
        sink.append(_quote(node))
        return
    if isinstance(node, dict):
        order = sorted(node) if sort_keys else list(node)
        sink.append("{")
        first = True
        for key in order:
            if not first:
                sink.append(", ")
            first = False
            sink.append(_quote(str(key)))
            sink.append(": ")
            _render(node[key], sort_keys, sink)
        sink.append("}")
        return
    if isinstance(node, (list, tuple)):
        sink.append("[")
        for pos, item in enumerate(node):
            if pos:
                sink.append(", ")
            _render(item, sort_keys, sink)
        sink.append("]")
        return
    raise TypeError(f"cannot serialize {type(node).__name__}")


def dumps_canonical(obj: Any, *, sort_keys: bool) -> str:
    """Single-line canonical document terminated by a newline."""
    sink: list = []
    _render(obj, sort_keys, sink)
    sink.append("\n")
    return "".join(sink)
