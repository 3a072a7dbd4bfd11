"""oracle/oracle.py — ctypes binding of the C oracle (oracle/gls_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  The product package never
imports this module.  It shares no code with the CUDA path.

`simulate()` runs Algorithm 2 gate by gate in topological
order and returns every net's waveform as a canonical CSR (packed
``(t << 2) | v`` entries, nets 0..P-1 = given waveforms verbatim, P+g = gate g).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gls_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C, -O2, single thread)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        vp = ctypes.c_void_p
        lib.oracle_simulate.restype = ctypes.c_int
        lib.oracle_simulate.argtypes = [ctypes.c_int32, ctypes.c_int32, vp, vp, vp, vp, vp, vp,
                                        ctypes.c_int64, ctypes.POINTER(vp)]
        lib.oracle_total.restype = ctypes.c_int64
        lib.oracle_total.argtypes = [vp]
        lib.oracle_stats.restype = None
        lib.oracle_stats.argtypes = [vp, vp]
        lib.oracle_get.restype = None
        lib.oracle_get.argtypes = [vp, vp, vp]
        lib.oracle_hashes.restype = None
        lib.oracle_hashes.argtypes = [vp, vp]
        lib.oracle_free.restype = None
        lib.oracle_free.argtypes = [vp]
        lib.oracle_simulate_cells.restype = ctypes.c_int
        lib.oracle_simulate_cells.argtypes = [ctypes.c_int32, ctypes.c_int32] + [vp] * 9 + [ctypes.c_int32, vp, vp, vp,
                                                                                          vp, vp, ctypes.c_int64,
                                                                                          ctypes.POINTER(vp)]
        lib.oracle_eval_gate.restype = ctypes.c_int
        lib.oracle_eval_gate.argtypes = [ctypes.c_int, vp, ctypes.c_int]
        _lib = lib
    return _lib


class OracleError(RuntimeError):
    pass


@dataclass
class OracleResult:
    offsets: np.ndarray      # int64 [P+G+1]
    trans: np.ndarray        # uint64 packed (t<<2)|v
    hashes: np.ndarray       # uint64 [P+G]
    gate_evals: int
    events: int
    out_trans: int

    def wave(self, net: int) -> list[tuple[int, int]]:
        e = self.trans[self.offsets[net]:self.offsets[net + 1]]
        return [(int(x >> 2), int(x & 3)) for x in e]


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def simulate(num_inputs, gate_type, fanin_offsets, fanin_net, pin_delay,
             in_offsets, in_trans, duration, want_waves=True) -> OracleResult:
    lib = _load()
    gate_type = _c(gate_type, np.uint8)
    fanin_offsets = _c(fanin_offsets, np.int64)
    fanin_net = _c(fanin_net, np.int32)
    pin_delay = _c(pin_delay, np.uint32).reshape(-1)
    in_offsets = _c(in_offsets, np.int64)
    in_trans = _c(in_trans, np.uint64)
    G = int(gate_type.shape[0])
    h = ctypes.c_void_p()
    rc = lib.oracle_simulate(int(num_inputs), G, gate_type.ctypes.data, fanin_offsets.ctypes.data,
                             fanin_net.ctypes.data, pin_delay.ctypes.data, in_offsets.ctypes.data,
                             in_trans.ctypes.data, int(duration), ctypes.byref(h))
    if rc != 0:
        raise OracleError(f"oracle_simulate failed rc={rc}")
    try:
        n = int(num_inputs) + G
        st = np.zeros(3, np.int64)
        lib.oracle_stats(h, st.ctypes.data)
        hashes = np.zeros(n, np.uint64)
        lib.oracle_hashes(h, hashes.ctypes.data)
        if want_waves:
            total = lib.oracle_total(h)
            offs = np.zeros(n + 1, np.int64)
            tr = np.zeros(max(total, 1), np.uint64)
            lib.oracle_get(h, offs.ctypes.data, tr.ctypes.data)
            tr = tr[:total]
        else:
            offs = np.zeros(0, np.int64)
            tr = np.zeros(0, np.uint64)
    finally:
        lib.oracle_free(h)
    return OracleResult(offs, tr, hashes, int(st[0]), int(st[1]), int(st[2]))


def eval_gate(gate_type: int, values) -> int:
    lib = _load()
    v = np.ascontiguousarray(values, dtype=np.uint8)
    return int(lib.oracle_eval_gate(int(gate_type), v.ctypes.data, int(v.shape[0])))


DELAY_INF = 0xFFFFFFFF


def pack_templates(templates):
    """templates: list of dict(n_in, n_out, gates=[(type, [node, ...]), ...], outputs=[node, ...]);
    node ids 0..n_in-1 = cell inputs, n_in + j = gate j.  Returns the flat arrays of
    oracle_simulate_cells (and of gls_load_cells)."""
    nin = np.array([t["n_in"] for t in templates], np.int32)
    nout = np.array([t["n_out"] for t in templates], np.int32)
    ng = np.array([len(t["gates"]) for t in templates], np.int32)
    gate_off = np.zeros(len(templates) + 1, np.int32)
    gate_off[1:] = np.cumsum(ng)
    types, fanin_off, fanin, out_node = [], [], [], []
    out_off = np.zeros(len(templates) + 1, np.int32)
    for i, t in enumerate(templates):
        for ty, nodes in t["gates"]:
            fanin_off.append(len(fanin))
            types.append(ty)
            fanin.extend(nodes)
        fanin_off.append(len(fanin))
        out_node.extend(t["outputs"])
        out_off[i + 1] = len(out_node)
    return dict(nin=nin, nout=nout, ngates=ng, gate_off=gate_off[:-1].copy(),
                gate_type=np.array(types or [0], np.uint8), fanin_off=np.array(fanin_off, np.int32),
                fanin=np.array(fanin or [0], np.int32), out_off=out_off[:-1].copy(),
                out_node=np.array(out_node or [0], np.int32))


def simulate_cells(num_inputs, templates, cell_tpl, cell_fanin, cell_delay, in_offsets, in_trans, duration,
                   want_waves=True) -> OracleResult:
    """Cell netlist (multi-output cells, UDP templates, DELAY_INF = no relation): nets
    0..P-1 given, then every cell's outputs in cell order.  cell_delay: per cell the
    [n_in][n_out][2 edge (RISE, FALL)][2 value (0, 1)] block, concatenated."""
    lib = _load()
    tp = pack_templates(templates)
    cell_tpl = _c(cell_tpl, np.int32)
    cell_fanin = _c(cell_fanin, np.int32)
    cell_delay = _c(cell_delay, np.uint32).reshape(-1)
    n_in = sum(templates[t]["n_in"] for t in cell_tpl)
    if cell_fanin.size != n_in or cell_delay.size != sum(4 * templates[t]["n_in"] * templates[t]["n_out"]
                                                          for t in cell_tpl):
        raise OracleError("cell_fanin / cell_delay sizes do not match the cells' templates")
    in_offsets = _c(in_offsets, np.int64)
    in_trans = _c(in_trans, np.uint64)
    h = ctypes.c_void_p()
    rc = lib.oracle_simulate_cells(int(num_inputs), len(templates), tp["nin"].ctypes.data, tp["nout"].ctypes.data,
                                   tp["ngates"].ctypes.data, tp["gate_off"].ctypes.data, tp["gate_type"].ctypes.data,
                                   tp["fanin_off"].ctypes.data, tp["fanin"].ctypes.data, tp["out_off"].ctypes.data,
                                   tp["out_node"].ctypes.data, int(cell_tpl.shape[0]), cell_tpl.ctypes.data,
                                   cell_fanin.ctypes.data, cell_delay.ctypes.data, in_offsets.ctypes.data,
                                   in_trans.ctypes.data if in_trans.size else None, int(duration), ctypes.byref(h))
    if rc != 0:
        raise OracleError(f"oracle_simulate_cells failed rc={rc}")
    try:
        n = int(num_inputs) + int(sum(templates[t]["n_out"] for t in cell_tpl))
        st = np.zeros(3, np.int64)
        lib.oracle_stats(h, st.ctypes.data)
        hashes = np.zeros(n, np.uint64)
        lib.oracle_hashes(h, hashes.ctypes.data)
        total = lib.oracle_total(h)
        offs = np.zeros(n + 1, np.int64)
        tr = np.zeros(max(total, 1), np.uint64)
        lib.oracle_get(h, offs.ctypes.data, tr.ctypes.data)
        tr = tr[:total]
    finally:
        lib.oracle_free(h)
    return OracleResult(offs, tr, hashes, int(st[0]), int(st[1]), int(st[2]))
