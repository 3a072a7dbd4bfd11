"""VCD front and back end (NEXT-4): stimulus import and result export.

The paper re-simulates from recorded waveform files ("WLF/VCD/FSDB") and its
problem statement takes the given waveforms of the primary / pseudo-primary inputs as
input.  `read_vcd` turns a Value Change Dump into the library's given-waveform
CSR (GLS_PACK entries, per-net strictly increasing times, no repeated value, a first value
of X dropped because every net starts at X — reading R6); `write_vcd` dumps the canonical
CSR of gls_get_waveforms.  Scalar signals and bit-blasted vectors (name[i]); values
0 / 1 / x / z; any $timescale (converted to ps).  Host-side I/O, not the hot path.
"""
from __future__ import annotations

import io
import re

import numpy as np

_VAL = {"0": 0, "1": 1, "x": 2, "X": 2, "z": 3, "Z": 3}
_CH = "0123"
_UNITS = {"s": 10 ** 12, "ms": 10 ** 9, "us": 10 ** 6, "ns": 10 ** 3, "ps": 1, "fs": None}


def _timescale_ps(text: str) -> int:
    m = re.match(r"\s*(\d+)\s*(s|ms|us|ns|ps|fs)\s*$", text)
    if not m or _UNITS[m.group(2)] is None:
        raise ValueError(f"unsupported $timescale {text!r} (integer ps resolution required)")
    return int(m.group(1)) * _UNITS[m.group(2)]


def read_vcd(src, input_names):
    """Parse a VCD (path, text or file object) into given waveforms for `input_names`
    (net order).  Returns (offsets int64 [P+1], transitions uint64 packed (t << 2) | v).
    Signals not in `input_names` are ignored; inputs absent from the dump stay X."""
    f = open(src) if isinstance(src, str) and "\n" not in src else (io.StringIO(src) if isinstance(src, str) else src)
    index = {n: i for i, n in enumerate(input_names)}
    ids = {}                                          # identifier -> [(pi, bit or None, width)]
    scale, t, scope = 1, 0, []
    waves = [dict() for _ in input_names]             # pi -> {time: value} (the last value at a time wins)
    in_defs = True
    tokens = f.read().split()
    i = 0
    while i < len(tokens):
        tok = tokens[i]
        if in_defs:
            if tok == "$timescale":
                j = tokens.index("$end", i)
                scale = _timescale_ps(" ".join(tokens[i + 1:j]))
                i = j + 1
                continue
            if tok == "$scope":
                scope.append(tokens[i + 2])
                i = tokens.index("$end", i) + 1
                continue
            if tok == "$upscope":
                scope.pop() if scope else None
                i = tokens.index("$end", i) + 1
                continue
            if tok == "$var":
                j = tokens.index("$end", i)
                width, code, name = int(tokens[i + 2]), tokens[i + 3], tokens[i + 4]
                rng = tokens[i + 5] if j > i + 5 else ""
                lo = 0
                m = re.match(r"\[(\d+):(\d+)\]", rng)
                if m:
                    lo = min(int(m.group(1)), int(m.group(2)))
                for cand in ([name] + [".".join(scope + [name])] if width == 1 and not m else []):
                    if cand in index:
                        ids.setdefault(code, []).append((index[cand], None, 1))
                if width > 1 or m:
                    for b in range(width):
                        for cand in (f"{name}[{lo + b}]", ".".join(scope + [f"{name}[{lo + b}]"])):
                            if cand in index:
                                ids.setdefault(code, []).append((index[cand], b, width))
                i = j + 1
                continue
            if tok == "$enddefinitions":
                in_defs = False
                i = tokens.index("$end", i) + 1
                continue
            i += 1
            continue
        if tok.startswith("#"):
            t = int(tok[1:]) * scale
        elif tok in ("$dumpvars", "$dumpall", "$dumpon", "$dumpoff", "$end"):
            pass
        elif tok[0] in "bB":
            bits, code = tok[1:], tokens[i + 1]
            i += 1
            for pi, b, width in ids.get(code, []):
                s = bits.rjust(width, "0" if bits[0] in "01" else bits[0])   # VCD left-extension
                waves[pi][t] = _VAL[s[width - 1 - b]]
        elif tok[0] in _VAL:
            for pi, _, _ in ids.get(tok[1:], []):
                waves[pi][t] = _VAL[tok[0]]
        i += 1
    offs = [0]
    trans = []
    for w in waves:
        prev = 2                                      # every net starts at X (R6)
        for tt in sorted(w):
            v = w[tt]
            if v != prev:
                trans.append((tt << 2) | v)
                prev = v
        offs.append(len(trans))
    return np.array(offs, np.int64), np.array(trans, np.uint64)


def _code(k: int) -> str:
    s = ""
    k += 1
    while k:
        k, r = divmod(k - 1, 94)
        s += chr(33 + r)
    return s


def write_vcd(dst, names, offsets, transitions, timescale="1ps", module="gls"):
    """Dump a waveform CSR (e.g. gls_get_waveforms) as VCD; `names` in net order.
    Initial values are X ($dumpvars), then every transition at its time."""
    offsets = np.asarray(offsets, np.int64)
    tr = np.asarray(transitions).view(np.uint64)
    n = len(offsets) - 1
    net = np.repeat(np.arange(n, dtype=np.int64), np.diff(offsets))
    t = (tr >> np.uint64(2)).astype(np.int64)
    v = (tr & np.uint64(3)).astype(np.int64)
    order = np.lexsort((net, t))
    out = open(dst, "w") if isinstance(dst, str) else dst
    try:
        out.write(f"$timescale {timescale} $end\n$scope module {module} $end\n")
        for k, nm in enumerate(names):
            out.write(f"$var wire 1 {_code(k)} {nm} $end\n")
        out.write("$upscope $end\n$enddefinitions $end\n#0\n$dumpvars\n")
        out.write("".join(f"x{_code(k)}\n" for k in range(n)))
        out.write("$end\n")
        cur = None
        for j in order:
            if t[j] != cur:
                cur = int(t[j])
                out.write(f"#{cur}\n")
            out.write(f"{'01xz'[v[j]]}{_code(int(net[j]))}\n")
    finally:
        if isinstance(dst, str):
            out.close()
