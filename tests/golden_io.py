"""Parsers for the text fixtures in tests/golden/ (test-only)."""
from __future__ import annotations

import os

from paper_2304_13398_b200 import workloads as W

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
VAL = {"0": 0, "1": 1, "x": 2, "X": 2, "z": 3, "Z": 3}


def table1():
    rows = []
    with open(os.path.join(GOLDEN, "table1.txt")) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            op, a, b, r = line.split()
            rows.append((op, VAL[a], VAL[b], VAL[r]))
    return rows


class Example:
    def __init__(self, name, cite):
        self.name, self.cite = name, cite
        self.default_delay = 5
        self.gates = []        # (out, type, [ins], {pin: (r0,r1,f0,f1)} or {'*': ...})
        self.inputs = {}       # name -> [(t, v)]
        self.duration = 100
        self.expect = {}       # name -> [(t, v)]

    def _tv(self, toks):
        out = []
        for tok in toks:
            t, v = tok.split(":")
            out.append((int(t), VAL[v]))
        return out

    def build(self):
        """-> (Netlist, Stimuli, duration, {net name: index}, expect {index: wave})."""
        in_names = list(self.inputs)
        index = {n: i for i, n in enumerate(in_names)}
        for g, (out, _, _, _) in enumerate(self.gates):
            index[out] = len(in_names) + g
        gates = []
        for out, typ, ins, dl in self.gates:
            dd = []
            for pin in ins:
                if pin in dl:
                    dd.append(dl[pin])
                elif "*" in dl:
                    dd.append(dl["*"])
                else:
                    dd.append((self.default_delay,) * 4)
            gates.append((W.TYPE_NAMES.index(typ), [index[p] for p in ins], dd))
        nl = W.netlist_from_gates(len(in_names), gates, list(index))
        st = W.stimuli_from_lists([self.inputs[n] for n in in_names])
        exp = {index[n]: w for n, w in self.expect.items()}
        return nl, st, self.duration, index, exp


def examples():
    exs, cur = [], None
    with open(os.path.join(GOLDEN, "examples.txt")) as f:
        for raw in f:
            line = raw.split("#", 1)[0].strip()
            if not line:
                continue
            toks = line.split()
            kw = toks[0]
            if kw == "example":
                cur = Example(toks[1], " ".join(toks[2:]))
                exs.append(cur)
            elif kw == "default_delay":
                cur.default_delay = int(toks[1])
            elif kw == "gate":
                body, _, dspec = line.partition(";")
                b = body.split()
                dl = {}
                for item in dspec.split():
                    pin, vals = item.split("=")
                    dl[pin] = tuple(int(x) for x in vals.split(","))
                cur.gates.append((b[1], b[2], b[3:], dl))
            elif kw == "input":
                cur.inputs[toks[1]] = cur._tv(toks[2:])
            elif kw == "duration":
                cur.duration = int(toks[1])
            elif kw == "expect":
                cur.expect[toks[1]] = cur._tv(toks[2:])
            else:
                raise ValueError(raw)
    return exs
