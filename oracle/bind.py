"""ctypes bindings of the CHECKERS (test infrastructure only).

* ``Oracle``    — liboracle.so, the plain-C restatement (pp_oracle.c).
* ``Reference`` — _ref/libpipeplan_ref.so, the unmodified reference planner
  (/root/reference/proj/src/*.cpp) behind ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm import this module.  Both expose ``plan(samples, grid, model, ...)`` and
``plan_tables(T, M, n, ...)`` returning the same ``Plan`` record the product
binding returns, so parity checks compare like with like.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpipeplan_ref.so")
REF_SRC = "/root/reference/proj"

PP_OK, PP_ERR_INVALID, PP_ERR_INFEASIBLE_SAMPLE, PP_ERR_INFEASIBLE = 0, 1, 2, 3


def build(ref: bool = True) -> None:
    """make liboracle.so (always) and _ref/ (when the reference tree exists)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref and os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def reference_available() -> bool:
    return os.path.exists(REF_SO)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class _GridDesc(C.Structure):
    _fields_ = [("n_mbs", C.c_int32), ("n_seq", C.c_int32), ("mbs_axis", C.c_void_p),
                ("seq_axis", C.c_void_p), ("cells", C.c_void_p)]


class _ModelDesc(C.Structure):
    _fields_ = [("n_stages", C.c_int32), ("encoder_layers", C.c_void_p),
                ("decoder_layers", C.c_void_p), ("is_encoder_decoder", C.c_int32),
                ("recompute", C.c_int32)]


class _Opts(C.Structure):
    _fields_ = [("stage_count", C.c_int32), ("replica_count", C.c_int32),
                ("per_mb_mem_cap", C.c_double), ("t_max_interval", C.c_double)]


def grid_desc(grid):
    mb = np.ascontiguousarray(grid.mbs_axis, np.int64)
    sq = np.ascontiguousarray(grid.seq_axis, np.int64)
    ce = np.ascontiguousarray(grid.cells, np.float64)
    return _GridDesc(len(mb), len(sq), _p(mb), _p(sq), _p(ce)), (mb, sq, ce)


def model_desc(model):
    enc = np.ascontiguousarray(model.encoder_layers, np.int32)
    dec = np.ascontiguousarray(model.decoder_layers, np.int32)
    return _ModelDesc(len(enc), _p(enc), _p(dec), int(model.is_encoder_decoder),
                      int(model.recompute)), (enc, dec)


class CheckerPlan:
    def __init__(self, status, splits=None, mb_times=None, t_max_used=math.nan,
                 objective=math.nan, err_sample_id=-1, ordered=None, n_candidates=-1,
                 n_evaluated=-1, replica=None, max_load=math.nan):
        self.status = status
        self.splits = splits
        self.mb_times = mb_times
        self.t_max_used = t_max_used
        self.objective = objective
        self.err_sample_id = err_sample_id
        self.ordered = ordered
        self.n_candidates = n_candidates
        self.n_evaluated = n_evaluated
        self.replica = replica
        self.max_load = max_load


class Oracle:
    """The C restatement."""

    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        L = C.CDLL(ORACLE_SO)
        vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
        L.orc_order_samples.argtypes = [vp, i64, vp]
        L.orc_per_layer.argtypes = [C.POINTER(_GridDesc), i32, i32, dbl, dbl, vp]
        L.orc_slice_cost.argtypes = [C.POINTER(_GridDesc), C.POINTER(_ModelDesc), vp, i64, i64, vp, vp]
        L.orc_dp_tables.argtypes = [vp, vp, i64, C.POINTER(_Opts), vp, vp, vp, vp, vp, vp, vp, vp]
        L.orc_plan_grid.argtypes = [vp, i64, i32, C.POINTER(_GridDesc), C.POINTER(_ModelDesc),
                                    C.POINTER(_Opts), vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.orc_plan_grid_stream.argtypes = [vp, i64, i32, C.POINTER(_GridDesc), C.POINTER(_ModelDesc),
                                           C.POINTER(_Opts), i32, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.orc_eval_objective.argtypes = [vp, i64, i32, i32, vp]
        L.orc_slice_extrema.argtypes = [vp, i64, C.POINTER(_GridDesc), C.POINTER(_ModelDesc), dbl,
                                        vp, vp]
        self.L = L

    def slice_extrema(self, ordered, grid, model, mem_cap=math.inf):
        """(max memory-feasible slice time, max singleton act_mem)."""
        o = np.ascontiguousarray(ordered, np.int64).reshape(-1, 3)
        g, k1 = grid_desc(grid)
        m, k2 = model_desc(model)
        t, a = np.zeros(1), np.zeros(1)
        self.L.orc_slice_extrema(_p(o), len(o), C.byref(g), C.byref(m), mem_cap, _p(t), _p(a))
        return float(t[0]), float(a[0])

    def order_samples(self, samples):
        s = np.ascontiguousarray(samples, np.int64).reshape(-1, 3)
        out = np.empty_like(s)
        rc = self.L.orc_order_samples(_p(s), len(s), _p(out))
        if rc != PP_OK:
            raise ValueError("mini-batch is empty")
        return out

    def per_layer(self, grid, kind, r, mbs, seq):
        g, keep = grid_desc(grid)
        out = np.zeros(3)
        self.L.orc_per_layer(C.byref(g), kind, r, float(mbs), float(seq), _p(out))
        return out

    def slice_cost(self, grid, model, ordered, begin, end):
        g, k1 = grid_desc(grid)
        m, k2 = model_desc(model)
        o = np.ascontiguousarray(ordered, np.int64)
        t, a = np.zeros(1), np.zeros(1)
        self.L.orc_slice_cost(C.byref(g), C.byref(m), _p(o), begin, end, _p(t), _p(a))
        return float(t[0]), float(a[0])

    def eval_objective(self, times, c, d):
        t = np.ascontiguousarray(times, np.float64)
        out = np.zeros(1)
        rc = self.L.orc_eval_objective(_p(t), len(t), c, d, _p(out))
        if rc != PP_OK:
            raise ValueError("bad objective arguments")
        return float(out[0])

    def plan_tables(self, T, M, n, stage_count, replica_count=1, mem_cap=math.inf,
                    t_max_interval=5.0):
        T = np.ascontiguousarray(T, np.float64)
        M = np.ascontiguousarray(M, np.float64)
        sp = np.zeros(max(n, 1), np.int32)
        tt = np.zeros(max(n, 1))
        cnt = np.zeros(1, np.int32)
        tm, ob = np.zeros(1), np.zeros(1)
        err = np.full(1, -1, np.int64)
        nc = np.zeros(1, np.int64)
        ne = np.zeros(1, np.int64)
        o = _Opts(stage_count, replica_count, mem_cap, t_max_interval)
        rc = self.L.orc_dp_tables(_p(T), _p(M), n, C.byref(o), _p(sp), _p(tt), _p(cnt), _p(tm),
                                  _p(ob), _p(err), _p(nc), _p(ne))
        if rc != PP_OK:
            return CheckerPlan(rc, err_sample_id=int(err[0]))
        m = int(cnt[0])
        return CheckerPlan(PP_OK, sp[:m].copy(), tt[:m].copy(), float(tm[0]), float(ob[0]),
                           n_candidates=int(nc[0]), n_evaluated=int(ne[0]))

    def plan(self, samples, grid, model, stage_count, replica_count=1, mem_cap=math.inf,
             t_max_interval=5.0, presorted=False):
        s = np.ascontiguousarray(samples, np.int64).reshape(-1, 3)
        n = len(s)
        g, k1 = grid_desc(grid)
        m, k2 = model_desc(model)
        o = _Opts(stage_count, replica_count, mem_cap, t_max_interval)
        ordered = np.empty_like(s)
        sp = np.zeros(max(n, 1), np.int32)
        tt = np.zeros(max(n, 1))
        cnt = np.zeros(1, np.int32)
        tm, ob = np.zeros(1), np.zeros(1)
        err = np.full(1, -1, np.int64)
        nc = np.zeros(1, np.int64)
        ne = np.zeros(1, np.int64)
        rc = self.L.orc_plan_grid(_p(s), n, int(presorted), C.byref(g), C.byref(m), C.byref(o),
                                  _p(ordered), _p(sp), _p(tt), _p(cnt), _p(tm), _p(ob), _p(err),
                                  _p(nc), _p(ne))
        if rc != PP_OK:
            return CheckerPlan(rc, err_sample_id=int(err[0]), ordered=ordered)
        k = int(cnt[0])
        return CheckerPlan(PP_OK, sp[:k].copy(), tt[:k].copy(), float(tm[0]), float(ob[0]),
                           ordered=ordered, n_candidates=int(nc[0]), n_evaluated=int(ne[0]))

    def plan_stream(self, samples, grid, model, stage_count, replica_count=1, mem_cap=math.inf,
                    t_max_interval=5.0, presorted=False, threads=None):
        """The streaming restatement (pp_stream.c): same record as plan(), no
        O(n^2) tables, `threads` OpenMP threads (default: all cores)."""
        s = np.ascontiguousarray(samples, np.int64).reshape(-1, 3)
        n = len(s)
        g, k1 = grid_desc(grid)
        m, k2 = model_desc(model)
        o = _Opts(stage_count, replica_count, mem_cap, t_max_interval)
        ordered = np.empty_like(s)
        sp = np.zeros(max(n, 1), np.int32)
        tt = np.zeros(max(n, 1))
        cnt = np.zeros(1, np.int32)
        tm, ob = np.zeros(1), np.zeros(1)
        err = np.full(1, -1, np.int64)
        nc = np.zeros(1, np.int64)
        ne = np.zeros(1, np.int64)
        rc = self.L.orc_plan_grid_stream(_p(s), n, int(presorted), C.byref(g), C.byref(m), C.byref(o),
                                         int(threads or os.cpu_count() or 1), _p(ordered), _p(sp), _p(tt),
                                         _p(cnt), _p(tm), _p(ob), _p(err), _p(nc), _p(ne))
        if rc != PP_OK:
            return CheckerPlan(rc, err_sample_id=int(err[0]), ordered=ordered)
        k = int(cnt[0])
        return CheckerPlan(PP_OK, sp[:k].copy(), tt[:k].copy(), float(tm[0]), float(ob[0]),
                           ordered=ordered, n_candidates=int(nc[0]), n_evaluated=int(ne[0]))


class RefGrid:
    """A grid built by the reference (fields as grid_desc reads them)."""

    def __init__(self, mbs_axis, seq_axis, cells):
        self.mbs_axis, self.seq_axis, self.cells = mbs_axis, seq_axis, cells


class RefModel:
    def __init__(self, enc, dec, encdec, recompute):
        self.encoder_layers, self.decoder_layers = enc, dec
        self.is_encoder_decoder, self.recompute = encdec, recompute


PADDING_ROW = np.dtype([("method", np.int32), ("reserved", np.int32), ("max_seq_len", np.int64),
                        ("padding_eff_input", np.float64), ("padding_eff_target", np.float64),
                        ("tokens", np.int64), ("sim_time", np.float64), ("throughput_proxy", np.float64)])


class Reference:
    """The unmodified reference planner (compiled from /root/reference)."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference at build time)")
        L = C.CDLL(REF_SO)
        vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
        L.ref_order_samples.argtypes = [vp, i64, vp]
        L.ref_per_layer.argtypes = [C.POINTER(_GridDesc), i32, i32, dbl, dbl, vp]
        L.ref_synthetic_grid.argtypes = [vp, i32, vp, i32, vp, i32, vp, vp, vp, vp]
        L.ref_load_dataset.argtypes = [i64, vp, vp, i64, C.c_uint64, vp]
        L.ref_model_uniform.argtypes = [i32, i32, i64, i32, vp, vp]
        L.ref_default_grid_params.argtypes = [vp, vp]
        L.ref_plan_grid.argtypes = [vp, i64, i32, C.POINTER(_GridDesc), C.POINTER(_ModelDesc),
                                    C.POINTER(_Opts), vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.ref_plan_tables.argtypes = [vp, vp, i64, C.POINTER(_Opts), vp, vp, vp, vp, vp, vp, vp, vp]
        L.ref_plan_batch.argtypes = [vp, vp, i32, C.POINTER(_GridDesc), C.POINTER(_ModelDesc),
                                     C.POINTER(_Opts), i32, vp, vp, vp, vp]
        L.ref_plan_batch.restype = dbl
        L.ref_plan_batch_out.argtypes = [vp, vp, i32, C.POINTER(_GridDesc), C.POINTER(_ModelDesc),
                                         C.POINTER(_Opts), i32, vp, vp, vp, vp, vp, vp, vp]
        L.ref_plan_batch_out.restype = dbl
        L.ref_op_costs.argtypes = [vp, i64, C.POINTER(_GridDesc), C.POINTER(_ModelDesc), vp, vp, vp]
        L.ref_emit_plans.argtypes = [vp, vp, vp, vp, i32, i32, vp, dbl, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                     vp, C.POINTER(_ModelDesc), i64, i32, i64, C.c_char_p, i64]
        L.ref_select_recomputation.argtypes = [vp, vp, i32, C.POINTER(_GridDesc), C.POINTER(_ModelDesc), i32, vp,
                                               vp, vp, vp, vp, vp]
        L.ref_order_search.argtypes = [vp, vp, vp, vp, i32, i32, vp, i32, dbl, i32, vp, vp, vp, vp, vp, vp]
        L.ref_order_search.restype = dbl
        L.ref_load_record_file.argtypes = [C.c_char_p, i64, vp, i64, vp, vp, vp, vp]
        L.ref_draw_all.argtypes = [vp, i64, i64, vp, vp]
        L.ref_padding_report.argtypes = [vp, i64, vp, i32, C.POINTER(_GridDesc), C.POINTER(_ModelDesc), i64,
                                         dbl, i32, i32, vp]
        L.ref_padding_report.restype = dbl
        self.L = L

    def order_samples(self, samples):
        s = np.ascontiguousarray(samples, np.int64).reshape(-1, 3)
        out = np.empty_like(s)
        rc = self.L.ref_order_samples(_p(s), len(s), _p(out))
        if rc != PP_OK:
            raise ValueError("mini-batch is empty")
        return out

    def per_layer(self, grid, kind, r, mbs, seq):
        g, keep = grid_desc(grid)
        out = np.zeros(3)
        self.L.ref_per_layer(C.byref(g), kind, r, float(mbs), float(seq), _p(out))
        return out

    def op_costs(self, shapes, grid, model):
        """The reference's OpCostTable::from_shapes -> (t_f, t_b, act), (n, stages)."""
        sh = np.ascontiguousarray(shapes, np.int64).reshape(-1, 3)
        g, k1 = grid_desc(grid)
        m, k2 = model_desc(model)
        C_ = len(model.encoder_layers)
        tf, tb, act = (np.zeros((len(sh), C_)) for _ in range(3))
        rc = self.L.ref_op_costs(_p(sh), len(sh), C.byref(g), C.byref(m), _p(tf), _p(tb), _p(act))
        if rc != PP_OK:
            raise ValueError(f"reference from_shapes failed: {rc}")
        return tf, tb, act

    def emit_plans(self, t_f, t_b, act_mem, mb_offset, limits=None, order=None, comm_latency=0.0,
                   one_f_one_b=False, shapes=None, model=None, iteration=0, replica=0, hidden=1024):
        """The reference's plan per table for the given order (or 1F1B):
        dict like capi.Planner.emit_plans plus "peers" and, with shapes and
        model, "plan_text" = save_plan of table 0."""
        tf = np.ascontiguousarray(t_f, np.float64)
        C_ = tf.shape[1]
        tb = np.ascontiguousarray(t_b, np.float64)
        ac = np.ascontiguousarray(act_mem, np.float64)
        off = np.ascontiguousarray(mb_offset, np.int64)
        S = len(off) - 1
        rows = int(off[-1])
        ins = np.zeros(max(rows, 1) * 10 * C_, np.int32)
        peer = np.zeros_like(ins)
        nins = np.zeros((S, C_), np.int32)
        ms, bub = np.zeros(S), np.zeros(S)
        dl, st = np.zeros(S, np.int32), np.zeros(S, np.int32)
        ds = np.zeros((S, C_, 5))
        lim = np.ascontiguousarray(limits if limits is not None else np.zeros(C_), np.float64)
        od = np.ascontiguousarray(order if order is not None else np.zeros(max(rows, 1)), np.int32)
        sh = np.ascontiguousarray(shapes if shapes is not None else np.zeros((1, 3)), np.int64)
        text = C.create_string_buffer(1 << 24)
        mdesc = None
        if model is not None:
            mdesc, _keep = model_desc(model)
        rc = self.L.ref_emit_plans(_p(tf), _p(tb), _p(ac), _p(off), S, C_, _p(lim), comm_latency,
                                   1 if one_f_one_b else 0, _p(od) if order is not None else None, _p(ins), _p(peer),
                                   _p(nins), _p(ms), _p(bub), _p(dl), _p(ds), _p(st),
                                   _p(sh) if shapes is not None else None,
                                   C.byref(mdesc) if mdesc is not None else None, iteration, replica, hidden, text,
                                   len(text))
        if rc != PP_OK:
            raise ValueError(f"reference emit failed: {rc}")
        lists, peers = [], []
        for s in range(S):
            m = int(off[s + 1] - off[s])
            per, pp_ = [], []
            for j in range(C_):
                o = 10 * C_ * off[s] + 10 * m * j
                a = ins[o:o + nins[s, j]]
                per.append(np.stack([a & 15, a >> 4], 1).astype(np.int32))
                pp_.append(peer[o:o + nins[s, j]].copy())
            lists.append(per)
            peers.append(pp_)
        return {"instructions": lists, "peers": peers, "makespan": ms, "bubble_ratio": bub, "deadlock": dl,
                "device_stats": ds, "status": st, "plan_text": text.value.decode()}

    def select_recomputation(self, shapes, mb_offset, grid, model, strategies=(0, 1, 2), limits=None):
        """The reference's select_recomputation per partition of shapes ->
        dict like capi.Planner.select_recomputation."""
        sh = np.ascontiguousarray(shapes, np.int64).reshape(-1, 3)
        off = np.ascontiguousarray(mb_offset, np.int64)
        g, k1 = grid_desc(grid)
        m, k2 = model_desc(model)
        S, C_ = len(off) - 1, len(model.encoder_layers)
        lim = np.ascontiguousarray(limits, np.float64)
        mask = sum(1 << int(r) for r in strategies)
        tf, tb, act = (np.zeros((max(len(sh), 1), C_)) for _ in range(3))
        st, vs = np.zeros(S, np.int32), np.zeros(S, np.int32)
        rc = self.L.ref_select_recomputation(_p(sh), _p(off), S, C.byref(g), C.byref(m), mask, _p(lim), _p(tf),
                                             _p(tb), _p(act), _p(st), _p(vs))
        if rc != PP_OK:
            raise ValueError(f"reference select_recomputation failed: {rc}")
        n = len(sh)
        return {"strategy": st, "violating_stage": vs, "t_f": tf[:n], "t_b": tb[:n], "act_mem": act[:n]}

    def order_search(self, t_f, t_b, act_mem, mb_offset, limits, n_clusters=3, comm_latency=0.0,
                     threads=1):
        """The reference's order_microbatches + the chosen order's SimReport
        (planner.cpp:94-108) per table; returns (wall seconds, dict)."""
        tf = np.ascontiguousarray(t_f, np.float64)
        tb = np.ascontiguousarray(t_b, np.float64)
        ac = np.ascontiguousarray(act_mem, np.float64)
        off = np.ascontiguousarray(mb_offset, np.int64)
        lim = np.ascontiguousarray(limits, np.float64)
        S, C_ = len(off) - 1, tf.shape[1]
        out = {"order": np.full(len(tf), -1, np.int32), "makespan": np.zeros(S), "bubble_ratio": np.zeros(S),
               "deadlock": np.zeros(S, np.int32), "device_stats": np.zeros((S, C_, 5)),
               "status": np.zeros(S, np.int32)}
        secs = self.L.ref_order_search(_p(tf), _p(tb), _p(ac), _p(off), S, C_, _p(lim), n_clusters,
                                       float(comm_latency), threads, _p(out["order"]), _p(out["makespan"]),
                                       _p(out["bubble_ratio"]), _p(out["deadlock"]), _p(out["device_stats"]),
                                       _p(out["status"]))
        return secs, out

    def load_record_file(self, path, max_seq_len, cap=None):
        """The reference's load_dataset(DatasetSpec{path}) -> (status, samples,
        err_line, err_byte, err_kind)."""
        if cap is None:
            cap = os.path.getsize(path) // 2 + 1
        out = np.zeros((cap, 3), np.int64)
        n, el, eb = (np.zeros(1, np.int64) for _ in range(3))
        ek = np.zeros(1, np.int32)
        rc = self.L.ref_load_record_file(str(path).encode(), max_seq_len, _p(out), cap, _p(n), _p(el), _p(eb),
                                         _p(ek))
        return rc, out[:min(int(n[0]), cap)].copy(), int(el[0]), int(eb[0]), int(ek[0])

    def draw_all(self, samples, budget):
        s = np.ascontiguousarray(samples, np.int64).reshape(-1, 3)
        off = np.zeros(len(s) + 1, np.int64)
        m = np.zeros(1, np.int64)
        rc = self.L.ref_draw_all(_p(s), len(s), budget, _p(off), _p(m))
        return rc, off[:int(m[0]) + 1].copy()

    def padding_report(self, samples, max_seq_lens, grid, model, token_budget=65536, t_max_interval=5.0,
                       max_iterations=0, recompute=0):
        """The reference's padding_vs_packing_report -> (seconds, rows (3L, 8) float64 view)."""
        s = np.ascontiguousarray(samples, np.int64).reshape(-1, 3)
        lens = np.ascontiguousarray(max_seq_lens, np.int64)
        g, k1 = grid_desc(grid)
        m, k2 = model_desc(model)
        rows = np.zeros(3 * len(lens), PADDING_ROW)
        secs = self.L.ref_padding_report(_p(s), len(s), _p(lens), len(lens), C.byref(g), C.byref(m), token_budget,
                                         t_max_interval, max_iterations, recompute, rows.ctypes.data)
        return secs, rows

    def synthetic_grid_cells(self, params7, tp, mbs_axis=(), seq_axis=()):
        par = np.asarray(params7, np.float64)
        ma = np.asarray(mbs_axis, np.int64)
        sa = np.asarray(seq_axis, np.int64)
        om, os_ = np.zeros(64, np.int64), np.zeros(64, np.int64)
        sizes = np.zeros(2, np.int32)
        cells = np.zeros(18 * 64 * 64)
        rc = self.L.ref_synthetic_grid(_p(par), tp, _p(ma), len(ma), _p(sa), len(sa), _p(om),
                                       _p(os_), _p(sizes), _p(cells))
        if rc != PP_OK:
            raise ValueError("invalid synthetic grid")
        nm, ns = int(sizes[0]), int(sizes[1])
        return om[:nm].copy(), os_[:ns].copy(), cells[:18 * nm * ns].reshape(2, 3, nm, ns, 3).copy()

    def default_grid(self):
        """ProfileGrid::synthetic(SyntheticGridParams{}) with the default
        axes, built by the reference itself."""
        par = np.zeros(7)
        tp = np.zeros(1, np.int32)
        self.L.ref_default_grid_params(_p(par), _p(tp))
        mb, sq, cells = self.synthetic_grid_cells(par, int(tp[0]))
        return RefGrid(mb, sq, cells)

    def model_uniform(self, n_stages, layers_per_stage, encoder_decoder, recompute=0, hidden_dim=1024):
        """ModelConfig::uniform (cost_model.cpp:273-292) + the Recompute
        make_slice_cost is called with."""
        enc = np.zeros(n_stages, np.int32)
        dec = np.zeros(n_stages, np.int32)
        rc = self.L.ref_model_uniform(n_stages, layers_per_stage, hidden_dim, int(encoder_decoder), _p(enc),
                                      _p(dec))
        if rc != PP_OK:
            raise ValueError("invalid model")
        return RefModel(enc, dec, bool(encoder_decoder), int(recompute))

    def load_dataset(self, n, max_seq_len, seed, input_dist, target_dist=None):
        out = np.zeros((n, 3), np.int64)
        ind = np.asarray(input_dist, np.float64)
        tgd = None if target_dist is None else np.asarray(target_dist, np.float64)
        rc = self.L.ref_load_dataset(n, _p(ind), _p(tgd), max_seq_len, seed, _p(out))
        if rc != PP_OK:
            raise ValueError("invalid dataset spec")
        return out

    def plan(self, samples, grid, model, stage_count, replica_count=1, mem_cap=math.inf,
             t_max_interval=5.0, presorted=False):
        s = np.ascontiguousarray(samples, np.int64).reshape(-1, 3)
        n = len(s)
        g, k1 = grid_desc(grid)
        m, k2 = model_desc(model)
        o = _Opts(stage_count, replica_count, mem_cap, t_max_interval)
        ordered = np.empty_like(s)
        sp = np.zeros(max(n, 1), np.int32)
        tt = np.zeros(max(n, 1))
        rep = np.zeros(max(n, 1), np.int32)
        cnt = np.zeros(1, np.int32)
        tm, ob, ml = np.zeros(1), np.zeros(1), np.zeros(1)
        err = np.full(1, -1, np.int64)
        rc = self.L.ref_plan_grid(_p(s), n, int(presorted), C.byref(g), C.byref(m), C.byref(o),
                                  _p(ordered), _p(sp), _p(tt), _p(cnt), _p(tm), _p(ob), _p(ml),
                                  _p(rep), _p(err))
        if rc != PP_OK:
            return CheckerPlan(rc, err_sample_id=int(err[0]))
        k = int(cnt[0])
        return CheckerPlan(PP_OK, sp[:k].copy(), tt[:k].copy(), float(tm[0]), float(ob[0]),
                           ordered=ordered, replica=rep[:k].copy(), max_load=float(ml[0]))

    def plan_tables(self, T, M, n, stage_count, replica_count=1, mem_cap=math.inf,
                    t_max_interval=5.0):
        T = np.ascontiguousarray(T, np.float64)
        M = np.ascontiguousarray(M, np.float64)
        sp = np.zeros(max(n, 1), np.int32)
        tt = np.zeros(max(n, 1))
        rep = np.zeros(max(n, 1), np.int32)
        cnt = np.zeros(1, np.int32)
        tm, ob, ml = np.zeros(1), np.zeros(1), np.zeros(1)
        err = np.full(1, -1, np.int64)
        o = _Opts(stage_count, replica_count, mem_cap, t_max_interval)
        rc = self.L.ref_plan_tables(_p(T), _p(M), n, C.byref(o), _p(sp), _p(tt), _p(cnt), _p(tm),
                                    _p(ob), _p(ml), _p(rep), _p(err))
        if rc != PP_OK:
            return CheckerPlan(rc, err_sample_id=int(err[0]))
        k = int(cnt[0])
        return CheckerPlan(PP_OK, sp[:k].copy(), tt[:k].copy(), float(tm[0]), float(ob[0]),
                           replica=rep[:k].copy(), max_load=float(ml[0]))

    def plan_batch_timed(self, samples, seg_offsets, grid, model, stage_count, replica_count=1,
                         mem_cap=math.inf, t_max_interval=5.0, threads=1):
        """run_plan-style worker pool; returns (wall seconds, t_max, objective, count, status)."""
        s = np.ascontiguousarray(samples, np.int64).reshape(-1, 3)
        off = np.ascontiguousarray(seg_offsets, np.int64)
        S = len(off) - 1
        g, k1 = grid_desc(grid)
        m, k2 = model_desc(model)
        o = _Opts(stage_count, replica_count, mem_cap, t_max_interval)
        tm, ob = np.zeros(S), np.zeros(S)
        cnt, st = np.zeros(S, np.int32), np.zeros(S, np.int32)
        secs = self.L.ref_plan_batch(_p(s), _p(off), S, C.byref(g), C.byref(m), C.byref(o), threads,
                                     _p(tm), _p(ob), _p(cnt), _p(st))
        return secs, tm, ob, cnt, st

    def plan_batch_full(self, samples, seg_offsets, grid, model, stage_count, replica_count=1,
                        mem_cap=math.inf, t_max_interval=5.0, threads=1):
        """plan_batch_timed that also returns every plan: dict of flat
        arrays indexed like the device's pp_plan_out (splits / mb_times /
        ordered_ids at each segment's sample offset) + 'seconds' (the
        planning wall time only)."""
        s = np.ascontiguousarray(samples, np.int64).reshape(-1, 3)
        off = np.ascontiguousarray(seg_offsets, np.int64)
        S = len(off) - 1
        g, k1 = grid_desc(grid)
        m, k2 = model_desc(model)
        o = _Opts(stage_count, replica_count, mem_cap, t_max_interval)
        r = {"t_max_used": np.zeros(S), "objective": np.zeros(S), "count": np.zeros(S, np.int32),
             "status": np.zeros(S, np.int32), "splits": np.zeros(len(s), np.int32),
             "mb_times": np.zeros(len(s)), "ordered_ids": np.zeros(len(s), np.int64)}
        r["seconds"] = self.L.ref_plan_batch_out(
            _p(s), _p(off), S, C.byref(g), C.byref(m), C.byref(o), threads, _p(r["t_max_used"]),
            _p(r["objective"]), _p(r["count"]), _p(r["status"]), _p(r["splits"]), _p(r["mb_times"]),
            _p(r["ordered_ids"]))
        return r
