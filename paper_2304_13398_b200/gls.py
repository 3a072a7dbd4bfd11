"""Thin ctypes binding of libgls.so (include/gls.h).

Argument marshalling only: every step of the simulation runs in the library's
CUDA kernels.  There is no CPU fallback — importing this module on a machine
without the built library raises, and every call returns the library's status
(non-zero statuses raise GlsError).  Names follow the C ABI.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GLS_LIB") or os.path.join(_HERE, "libgls.so")

GLS_OK, GLS_EINVAL, GLS_ECYCLE, GLS_ENOMEM, GLS_ESTATE, GLS_ERANGE, GLS_ECUDA = 0, -1, -2, -3, -4, -5, -6
STATUS = {0: "GLS_OK", -1: "GLS_EINVAL", -2: "GLS_ECYCLE", -3: "GLS_ENOMEM", -4: "GLS_ESTATE",
          -5: "GLS_ERANGE", -6: "GLS_ECUDA"}

EXPORTS = ["gls_create", "gls_destroy", "gls_last_error", "gls_version", "gls_set_config",
           "gls_load_netlist", "gls_set_input_waveforms", "gls_set_input_waveforms_device",
           "gls_simulate", "gls_simulate_window", "gls_get_waveforms", "gls_get_net_hashes", "gls_get_net_hashes_device",
           "gls_get_net_hashes_window", "gls_get_net_hash_terms_device",
           "gls_get_net_counts", "gls_get_stats", "gls_get_halo", "gls_get_levels", "gls_lut_lookup",
           "gls_get_waveforms_range_device", "gls_scatter_segments", "gls_load_cells", "gls_get_trace"]

GLS_DELAY_INF = 0xFFFFFFFF


class GlsError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class gls_config(ctypes.Structure):
    _fields_ = [("arena_bytes", ctypes.c_int64), ("chunk_capacity", ctypes.c_int64),
                ("chunk_events", ctypes.c_int32), ("blocks_per_sm", ctypes.c_int32),
                ("ring_limit", ctypes.c_int32), ("engine", ctypes.c_int32), ("scheduler", ctypes.c_int32),
                ("deep_per_warp", ctypes.c_int64), ("readback_mib", ctypes.c_int32), ("trace", ctypes.c_int32),
                ("csrp_pagelen", ctypes.c_int32)]


class gls_cell_template(ctypes.Structure):
    _fields_ = [("num_inputs", ctypes.c_int32), ("num_outputs", ctypes.c_int32), ("num_gates", ctypes.c_int32),
                ("gate_type", ctypes.c_void_p), ("gate_fanin_offsets", ctypes.c_void_p),
                ("gate_fanin", ctypes.c_void_p), ("output_node", ctypes.c_void_p)]


class gls_stats(ctypes.Structure):
    _fields_ = [("gate_evals", ctypes.c_int64), ("events", ctypes.c_int64),
                ("out_transitions", ctypes.c_int64), ("chunks", ctypes.c_int64),
                ("deep_chunks", ctypes.c_int64), ("levels", ctypes.c_int64),
                ("arena_used_bytes", ctypes.c_int64), ("alg_bytes", ctypes.c_int64),
                ("fanin_reads", ctypes.c_int64),
                ("lane_utilization", ctypes.c_double), ("batches", ctypes.c_int64),
                ("batch_lanes", ctypes.c_double), ("batch_est", ctypes.c_double),
                ("phase_cycles", ctypes.c_double * 6), ("balance", ctypes.c_double * 8),
                ("kernel_ms", ctypes.c_double), ("csrp_pages", ctypes.c_int64), ("csrp_waste", ctypes.c_int64),
                ("simulate_ms", ctypes.c_double)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["phase_cycles"] = list(self.phase_cycles)
        d["balance"] = list(self.balance)
        return d


_lib = None


def load_library():
    """Load libgls.so (built in-tree by __graft_entry__.build() / make)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} not built: run `make` or __graft_entry__.build() (no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, p = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.POINTER
    sig = {
        "gls_create": (ctypes.c_int, [p(vp), ctypes.c_int, vp]),
        "gls_destroy": (None, [vp]),
        "gls_last_error": (ctypes.c_char_p, [vp]),
        "gls_version": (ctypes.c_char_p, []),
        "gls_set_config": (ctypes.c_int, [vp, p(gls_config)]),
        "gls_load_netlist": (ctypes.c_int, [vp, i32, i32, vp, vp, vp, vp]),
        "gls_set_input_waveforms": (ctypes.c_int, [vp, i32, vp, vp]),
        "gls_set_input_waveforms_device": (ctypes.c_int, [vp, i32, vp, vp, i64]),
        "gls_simulate": (ctypes.c_int, [vp, i64]),
        "gls_simulate_window": (ctypes.c_int, [vp, i64, i64, i64]),
        "gls_get_waveforms": (ctypes.c_int, [vp, vp, vp, i64, p(i64)]),
        "gls_get_net_hashes": (ctypes.c_int, [vp, vp]),
        "gls_get_net_hashes_device": (ctypes.c_int, [vp, vp]),
        "gls_get_net_hashes_window": (ctypes.c_int, [vp, i64, i64, vp]),
        "gls_get_net_hash_terms_device": (ctypes.c_int, [vp, i64, i64, vp, vp, vp, vp]),
        "gls_get_net_counts": (ctypes.c_int, [vp, vp]),
        "gls_get_stats": (ctypes.c_int, [vp, p(gls_stats)]),
        "gls_get_halo": (ctypes.c_int, [vp, p(i64)]),
        "gls_get_levels": (ctypes.c_int, [vp, p(i32)]),
        "gls_lut_lookup": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, vp]),
        "gls_get_waveforms_range_device": (ctypes.c_int, [vp, i64, i64, i64, i64, vp, vp, i64, p(i64)]),
        "gls_scatter_segments": (ctypes.c_int, [vp, i64, vp, vp, vp, vp]),
        "gls_load_cells": (ctypes.c_int, [vp, i32, i32, vp, i32, vp, vp, vp]),
        "gls_get_trace": (ctypes.c_int, [vp, vp]),
    }
    for name, (res, args) in sig.items():
        if os.environ.get("GLS_AB_OLD") and not hasattr(lib, name):
            continue                    # A/B against an older build of the library (experiments only)
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _arr(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def gls_version() -> str:
    return load_library().gls_version().decode()


def gls_lut_lookup(gate_type: int, arity: int, values) -> int:
    v = _arr(values, np.uint8)
    return int(load_library().gls_lut_lookup(int(gate_type), int(arity), v.ctypes.data))


@dataclass
class Waveforms:
    offsets: np.ndarray   # int64 [nets+1]
    trans: np.ndarray     # uint64 packed

    def wave(self, net):
        e = self.trans[self.offsets[net]:self.offsets[net + 1]]
        return [(int(x >> 2), int(x & 3)) for x in e]


class Context:
    """One gls_ctx.  `stream` is a cudaStream_t as int (e.g.
    torch.cuda.current_stream().cuda_stream) or None for the default stream."""

    def __init__(self, device: int = 0, stream: int | None = None):
        self._lib = load_library()
        h = ctypes.c_void_p()
        rc = self._lib.gls_create(ctypes.byref(h), int(device), ctypes.c_void_p(stream or 0))
        if rc != GLS_OK:
            raise GlsError(rc, "gls_create failed")
        self._h = h
        self._keep = []

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.gls_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _check(self, rc):
        if rc != GLS_OK:
            raise GlsError(rc, self._lib.gls_last_error(self._h).decode())
        return rc

    def last_error(self) -> str:
        return self._lib.gls_last_error(self._h).decode()

    # ---- ABI calls ----------------------------------------------------------
    def gls_set_config(self, arena_bytes=0, chunk_capacity=0, chunk_events=0, blocks_per_sm=0, ring_limit=0,
                       engine=0, scheduler=0, deep_per_warp=0, readback_mib=0, trace=0, csrp_pagelen=0):
        c = gls_config(arena_bytes, chunk_capacity, chunk_events, blocks_per_sm, ring_limit, engine, scheduler,
                       deep_per_warp, readback_mib, trace, csrp_pagelen)
        return self._check(self._lib.gls_set_config(self._h, ctypes.byref(c)))

    def gls_load_netlist(self, num_inputs, gate_type, fanin_offsets, fanin_net, pin_delay):
        gt = _arr(gate_type, np.uint8)
        fo = _arr(fanin_offsets, np.int64)
        fn = _arr(fanin_net, np.int32)
        pd = _arr(pin_delay, np.uint32).reshape(-1)
        self.num_inputs, self.num_gates = int(num_inputs), int(gt.shape[0])
        return self._check(self._lib.gls_load_netlist(self._h, int(num_inputs), int(gt.shape[0]),
                                                      gt.ctypes.data, fo.ctypes.data, fn.ctypes.data,
                                                      pd.ctypes.data))

    def gls_load_cells(self, num_inputs, templates, cell_template, cell_fanin, cell_delay):
        """templates: list of dict(n_in, n_out, gates=[(type, [node, ...]), ...], outputs=[node, ...])
        (node ids: 0..n_in-1 cell inputs, n_in + j gate j); cell_delay: per cell the
        [n_in][n_out][2 edge][2 value] block, concatenated (GLS_DELAY_INF = no relation)."""
        keep = []
        arr = (gls_cell_template * max(1, len(templates)))()
        for i, t in enumerate(templates):
            ty = _arr([g[0] for g in t["gates"]] or [0], np.uint8)
            fo = np.zeros(len(t["gates"]) + 1, np.int32)
            fo[1:] = np.cumsum([len(g[1]) for g in t["gates"]]) if t["gates"] else []
            fi = _arr([x for g in t["gates"] for x in g[1]] or [0], np.int32)
            on = _arr(t["outputs"], np.int32)
            keep += [ty, fo, fi, on]
            arr[i] = gls_cell_template(int(t["n_in"]), int(t["n_out"]), len(t["gates"]), ty.ctypes.data,
                                       fo.ctypes.data, fi.ctypes.data, on.ctypes.data)
        ct = _arr(cell_template, np.int32)
        cf = _arr(cell_fanin, np.int32)
        cd = _arr(cell_delay, np.uint32).reshape(-1)
        if (ct.size and (ct.min() < 0 or ct.max() >= len(templates))) or \
                cf.size != sum(templates[t]["n_in"] for t in ct) or \
                cd.size != sum(4 * templates[t]["n_in"] * templates[t]["n_out"] for t in ct):
            raise GlsError(GLS_EINVAL, "cell_template / cell_fanin / cell_delay do not match the templates")
        rc = self._lib.gls_load_cells(self._h, int(num_inputs), len(templates), ctypes.addressof(arr), int(ct.shape[0]),
                                      ct.ctypes.data, cf.ctypes.data, cd.ctypes.data)
        self.num_inputs = int(num_inputs)
        self.num_gates = int(sum(templates[t]["n_out"] for t in ct))
        return self._check(rc)

    def load(self, nl):
        return self.gls_load_netlist(nl.num_inputs, nl.gate_type, nl.fanin_offsets, nl.fanin_net, nl.pin_delay)

    def gls_set_input_waveforms(self, num_inputs, offsets, transitions):
        o = _arr(offsets, np.int64)
        t = _arr(transitions, np.uint64)
        return self._check(self._lib.gls_set_input_waveforms(self._h, int(num_inputs), o.ctypes.data,
                                                             t.ctypes.data if t.size else None))

    def gls_set_input_waveforms_device(self, num_inputs, d_offsets_ptr, d_trans_ptr, total):
        return self._check(self._lib.gls_set_input_waveforms_device(
            self._h, int(num_inputs), ctypes.c_void_p(d_offsets_ptr), ctypes.c_void_p(d_trans_ptr), int(total)))

    def gls_simulate(self, duration):
        return self._check(self._lib.gls_simulate(self._h, int(duration)))

    def gls_simulate_window(self, t_begin, t_end, duration):
        return self._check(self._lib.gls_simulate_window(self._h, int(t_begin), int(t_end), int(duration)))

    def gls_get_waveforms(self) -> Waveforms:
        n = self.num_inputs + self.num_gates
        total = ctypes.c_int64()
        offs = np.zeros(n + 1, np.int64)
        self._check(self._lib.gls_get_waveforms(self._h, offs.ctypes.data, None, 0, ctypes.byref(total)))
        tr = np.zeros(max(1, total.value), np.uint64)
        self._check(self._lib.gls_get_waveforms(self._h, offs.ctypes.data, tr.ctypes.data, tr.size,
                                                ctypes.byref(total)))
        return Waveforms(offs, tr[:total.value])

    def gls_get_waveforms_range_device(self, net_lo, net_hi, t_lo, t_hi, d_offsets, d_trans=0, capacity=0) -> int:
        """Device pointers (ints; d_trans 0 = size query).  Returns the transition count."""
        total = ctypes.c_int64()
        self._check(self._lib.gls_get_waveforms_range_device(
            self._h, int(net_lo), int(net_hi), int(t_lo), int(t_hi), ctypes.c_void_p(d_offsets),
            ctypes.c_void_p(d_trans) if d_trans else None, int(capacity), ctypes.byref(total)))
        return total.value

    def gls_scatter_segments(self, nseg, d_src_off, d_src, d_dst_off, d_dst):
        vp = lambda x: ctypes.c_void_p(x) if x else None
        return self._check(self._lib.gls_scatter_segments(self._h, int(nseg), vp(d_src_off), vp(d_src),
                                                          vp(d_dst_off), vp(d_dst)))

    def gls_get_net_hashes(self) -> np.ndarray:
        h = np.zeros(self.num_inputs + self.num_gates, np.uint64)
        self._check(self._lib.gls_get_net_hashes(self._h, h.ctypes.data))
        return h

    def gls_get_net_hashes_window(self, t_lo, t_hi) -> np.ndarray:
        h = np.zeros(self.num_inputs + self.num_gates, np.uint64)
        self._check(self._lib.gls_get_net_hashes_window(self._h, int(t_lo), int(t_hi), h.ctypes.data))
        return h

    def gls_get_net_hashes_device(self, d_ptr):
        return self._check(self._lib.gls_get_net_hashes_device(self._h, ctypes.c_void_p(d_ptr)))

    def gls_get_net_hash_terms_device(self, t_lo, t_hi, d_base, d_total, d_counts, d_terms):
        """Device pointers (ints, 0 = NULL): window stitching pieces (include/gls.h)."""
        vpn = lambda x: ctypes.c_void_p(x) if x else None
        return self._check(self._lib.gls_get_net_hash_terms_device(
            self._h, int(t_lo), int(t_hi), vpn(d_base), vpn(d_total), vpn(d_counts), vpn(d_terms)))

    def gls_get_net_counts(self) -> np.ndarray:
        c = np.zeros(self.num_inputs + self.num_gates, np.int64)
        self._check(self._lib.gls_get_net_counts(self._h, c.ctypes.data))
        return c

    def gls_get_stats(self) -> dict:
        s = gls_stats()
        self._check(self._lib.gls_get_stats(self._h, ctypes.byref(s)))
        return s.as_dict()

    def gls_get_trace(self) -> np.ndarray:
        t = np.zeros((self.num_gates, 8), np.uint64)
        self._check(self._lib.gls_get_trace(self._h, t.ctypes.data))
        return t

    def gls_get_halo(self) -> int:
        h = ctypes.c_int64()
        self._check(self._lib.gls_get_halo(self._h, ctypes.byref(h)))
        return h.value

    def gls_get_levels(self) -> int:
        h = ctypes.c_int32()
        self._check(self._lib.gls_get_levels(self._h, ctypes.byref(h)))
        return h.value


def simulate(nl, stim, duration, device=0, **config) -> tuple[Waveforms, dict]:
    """Convenience: one context, load, set inputs, simulate, read back."""
    with Context(device) as c:
        if config:
            c.gls_set_config(**config)
        c.load(nl)
        c.gls_set_input_waveforms(nl.num_inputs, stim.offsets, stim.trans)
        c.gls_simulate(duration)
        return c.gls_get_waveforms(), c.gls_get_stats()
