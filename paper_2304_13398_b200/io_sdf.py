"""SDF-like delay import (NEXT-4): IOPATH delays of gate instances into the
library's pin-to-pin delay array (§2.3; the 5-D matrix of §3.2).

Supported subset of SDF 3.0: (TIMESCALE n unit), (CELL (CELLTYPE ..) (INSTANCE name)
(DELAY (ABSOLUTE|INCREMENT (IOPATH in out rise [fall]) ...))), delay values as a number or
(min:typ:max) (the typical value is taken; a missing fall = rise), input pins optionally
qualified (posedge p) / (negedge p).  SDF delays are per OUTPUT edge: `rise` is the delay
of an output change to 1, `fall` to 0; without an edge qualifier they apply to both input
edges.  INCREMENT adds to the current value.  Host-side I/O, not the hot path.
"""
from __future__ import annotations

import re

import numpy as np

_SCALE = {"s": 10 ** 12, "ms": 10 ** 9, "us": 10 ** 6, "ns": 10 ** 3, "ps": 1}
DEFAULT_PINS = ["A", "B", "C", "D"]              # input pin names by position (MUX2: A, B, S)


def _parse(text):
    toks = re.findall(r'\(|\)|"[^"]*"|[^\s()]+', text)
    pos = 0

    def node():
        nonlocal pos
        if toks[pos] == "(":
            pos += 1
            out = []
            while toks[pos] != ")":
                out.append(node())
            pos += 1
            return out
        t = toks[pos]
        pos += 1
        return t.strip('"')
    return node()


def _value(v, scale):
    """number or [min:typ:max] / (typ) -> ps (float -> rounded int)"""
    if isinstance(v, list):
        v = v[0] if v else "0"
    parts = str(v).split(":")
    x = parts[1] if len(parts) == 3 and parts[1] else parts[0]
    return int(round(float(x) * scale))


def read_sdf(text, gate_names, fanin_offsets, pin_delay, gate_type=None, pin_names=None):
    """Apply the IOPATHs of an SDF text to `pin_delay` ([E][4] u32, (rise->0, rise->1,
    fall->0, fall->1) per pin, modified in place and returned).  gate_names: instance name
    of each gate; pin_names(g) -> input pin names of gate g in fan-in order (default A, B,
    C, D; MUX2 A, B, S).  Unknown instances / pins raise ValueError."""
    tree = _parse(text)
    if not tree or tree[0] != "DELAYFILE":
        raise ValueError("not an SDF DELAYFILE")
    gi = {n: g for g, n in enumerate(gate_names)}
    pin_delay = np.asarray(pin_delay, np.uint32).reshape(-1, 4)
    scale = 1
    for item in tree[1:]:
        if not isinstance(item, list) or not item:
            continue
        if item[0] == "TIMESCALE":
            m = re.match(r"(\d+(?:\.\d+)?)\s*(s|ms|us|ns|ps)$", "".join(item[1:]))
            if not m:
                raise ValueError(f"TIMESCALE {item[1:]}")
            scale = float(m.group(1)) * _SCALE[m.group(2)]
        if item[0] != "CELL":
            continue
        inst = next((x[1] for x in item if isinstance(x, list) and x and x[0] == "INSTANCE"), None)
        if inst not in gi:
            raise ValueError(f"unknown instance {inst!r}")
        g = gi[inst]
        k = int(fanin_offsets[g + 1] - fanin_offsets[g])
        names = pin_names(g) if pin_names else (["A", "B", "S"] if gate_type is not None and int(gate_type[g]) == 8
                                                 else DEFAULT_PINS[:k])
        for d in (x for x in item if isinstance(x, list) and x and x[0] == "DELAY"):
            for block in d[1:]:
                incr = block[0] == "INCREMENT"
                for path in block[1:]:
                    if not isinstance(path, list) or path[0] != "IOPATH":
                        continue
                    pin, edges = path[1], (0, 1)            # input edge RISE = 0, FALL = 1
                    if isinstance(pin, list):
                        edges = (0,) if pin[0] == "posedge" else (1,)
                        pin = pin[1]
                    if pin not in names:
                        raise ValueError(f"{inst}: unknown pin {pin!r}")
                    rise = _value(path[3], scale)
                    fall = _value(path[4], scale) if len(path) > 4 else rise
                    row = pin_delay[int(fanin_offsets[g]) + names.index(pin)]
                    for e in edges:
                        for val, dv in ((0, fall), (1, rise)):
                            c = e * 2 + val
                            row[c] = (int(row[c]) + dv) if incr else dv
    return pin_delay
