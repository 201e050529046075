"""ctypes binding of the B200 planner C-ABI (include/pipeplan_b200.h).

This is the Python face of the drop-in boundary: the same entry points a
cgo / JNI / ctypes caller of the reference planner would bind (see
INTEGRATION.md).  Arrays are numpy; samples are an (n, 3) int64 array of
(id, input_len, target_len) rows — the memory layout of pipeplan::Sample.

There is no CPU fallback anywhere below: if the shared library is missing the
import fails, and if no CUDA device is present ``Planner()`` raises
``NoDeviceError``.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field

import numpy as np

_LIB_PATH = os.environ.get("PIPEPLAN_B200_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libpipeplan_b200.so")

PP_OK, PP_ERR_INVALID, PP_ERR_INFEASIBLE_SAMPLE, PP_ERR_INFEASIBLE = 0, 1, 2, 3
PP_ERR_CUDA, PP_ERR_NO_DEVICE, PP_ERR_OUT_OF_RANGE = 4, 5, 6
PP_ERR_NOT_CONVERGED, PP_ERR_NOT_EXECUTABLE, PP_ERR_PARSE = 7, 8, 9

# Every symbol include/pipeplan_b200.h declares (checked by the CPU tests).
EXPORTED = [
    "pp_abi_version", "pp_ctx_create", "pp_ctx_destroy", "pp_ctx_last_error", "pp_ctx_set_tuning",
    "pp_ctx_get_stats", "pp_ctx_set_stream", "pp_order_samples", "pp_plan_grid",
    "pp_plan_grid_device", "pp_plan_tables", "pp_candidate_range", "pp_eval_objective",
    "pp_synthetic_grid", "pp_synthetic_dataset", "pp_slice_cost_host", "pp_calibrate_fp64",
    "pp_op_costs", "pp_plan_op_costs_device", "pp_order_search", "pp_order_search_device",
    "pp_load_records", "pp_load_records_device", "pp_draw_minibatches", "pp_draw_minibatches_device",
    "pp_padding_report", "pp_assign_replicas", "pp_pack_plan_slots", "pp_select_recomputation",
    "pp_select_recomputation_device", "pp_emit_plans", "pp_emit_plans_device", "pp_format_plan",
]


PADDING_ROW = np.dtype([("method", np.int32), ("reserved", np.int32), ("max_seq_len", np.int64),
                        ("padding_eff_input", np.float64), ("padding_eff_target", np.float64),
                        ("tokens", np.int64), ("sim_time", np.float64), ("throughput_proxy", np.float64)])


class PlannerError(RuntimeError):
    pass


class NoDeviceError(PlannerError):
    pass


class InvalidArgument(PlannerError, ValueError):
    pass


class ParseError(PlannerError, ValueError):
    """pipeplan::ParseError (errors.h:25-40): line (1-based), byte offset."""

    def __init__(self, msg: str, line: int, byte_offset: int, kind: int = -1):
        super().__init__(msg)
        self.line, self.byte_offset, self.kind = line, byte_offset, kind


class InfeasibleError(PlannerError):
    """Mirror of pipeplan::InfeasibleError (errors.h:43-56)."""

    def __init__(self, msg: str, sample_id: int = -1, stage: int = -1):
        super().__init__(msg)
        self.sample_id = sample_id
        self.stage = stage


# ----------------------------------------------------------------- structs
class GridDesc(C.Structure):
    _fields_ = [("n_mbs", C.c_int32), ("n_seq", C.c_int32), ("mbs_axis", C.c_void_p),
                ("seq_axis", C.c_void_p), ("cells", C.c_void_p)]


class ModelDesc(C.Structure):
    _fields_ = [("n_stages", C.c_int32), ("encoder_layers", C.c_void_p),
                ("decoder_layers", C.c_void_p), ("is_encoder_decoder", C.c_int32),
                ("recompute", C.c_int32)]


class DpOptions(C.Structure):
    _fields_ = [("stage_count", C.c_int32), ("replica_count", C.c_int32),
                ("per_mb_mem_cap", C.c_double), ("t_max_interval", C.c_double)]


class Tuning(C.Structure):
    _fields_ = [("first_wave", C.c_int32), ("max_wave", C.c_int32), ("streams", C.c_int32),
                ("coop_min_n", C.c_int32), ("no_slice_reuse", C.c_int32), ("no_band_trunc", C.c_int32),
                ("compact_band", C.c_int32), ("host_chunks", C.c_int32), ("dp_pricing", C.c_int32),
                ("no_slice_table", C.c_int32), ("no_bin_intervals", C.c_int32)]


class PlanOut(C.Structure):
    _fields_ = [("ordered", C.c_void_p), ("splits", C.c_void_p), ("mb_times", C.c_void_p),
                ("count", C.c_void_p), ("t_max_used", C.c_void_p), ("objective", C.c_void_p),
                ("status", C.c_void_p), ("err_sample_id", C.c_void_p), ("order", C.c_void_p)]


KERNEL_NAMES = ["segmented sort", "cost setup", "cost pass A (act_mem row widths)",
                "cost pass B (band tiles + candidate bins)", "DP bound pass (+ first candidate, fused)", "DP candidate passes",
                "candidate compaction", "selection / assembly"]


class Stats(C.Structure):
    _fields_ = [("candidates_generated", C.c_int64), ("candidates_evaluated", C.c_int64),
                ("transitions_executed", C.c_int64), ("transitions_reference", C.c_int64),
                ("slices_costed", C.c_int64), ("waves", C.c_int64), ("ms_sort", C.c_double),
                ("ms_cost", C.c_double), ("ms_dp", C.c_double), ("ms_total", C.c_double),
                ("ms_kernel", C.c_double * 8), ("launches", C.c_int64 * 8),
                ("dp_band_bytes", C.c_int64), ("slices_pass_a", C.c_int64),
                ("exit_thresh", C.c_double), ("slices_pass_b", C.c_int64),
                ("bound_transitions", C.c_int64), ("band_bytes", C.c_int64),
                ("candidates_ref_evaluated", C.c_int64)]

    def as_dict(self):
        out = {}
        for k, _ in self._fields_:
            v = getattr(self, k)
            out[k] = list(v) if k in ("ms_kernel", "launches") else v
        return out


def _load():
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} is missing: run __graft_entry__.build() "
                          "(the planner has no CPU fallback)")
    lib = C.CDLL(_LIB_PATH)
    vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    lib.pp_ctx_last_error.restype = C.c_char_p
    lib.pp_ctx_last_error.argtypes = [vp]
    lib.pp_ctx_create.argtypes = [C.c_int, C.POINTER(vp)]
    lib.pp_ctx_destroy.argtypes = [vp]
    lib.pp_ctx_set_tuning.argtypes = [vp, C.POINTER(Tuning)]
    lib.pp_ctx_get_stats.argtypes = [vp, C.POINTER(Stats)]
    lib.pp_ctx_set_stream.argtypes = [vp, vp]
    lib.pp_order_samples.argtypes = [vp, vp, vp, i32, vp]
    lib.pp_plan_grid.argtypes = [vp, vp, vp, i32, i32, C.POINTER(GridDesc), C.POINTER(ModelDesc),
                                 C.POINTER(DpOptions), C.POINTER(PlanOut)]
    lib.pp_plan_grid_device.argtypes = [vp, vp, vp, vp, i32, i32, C.POINTER(GridDesc),
                                        C.POINTER(ModelDesc), C.POINTER(DpOptions),
                                        C.POINTER(PlanOut)]
    lib.pp_plan_tables.argtypes = [vp, vp, vp, i64, C.POINTER(DpOptions), vp, vp, vp, vp, vp, vp]
    lib.pp_candidate_range.argtypes = [vp, vp, vp, i32, i32, C.POINTER(GridDesc),
                                       C.POINTER(ModelDesc), dbl, vp, vp]
    lib.pp_eval_objective.argtypes = [vp, i64, i32, i32, vp]
    lib.pp_assign_replicas.argtypes = [vp, i64, i32, vp, vp]
    lib.pp_pack_plan_slots.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, i32, i32, vp]
    lib.pp_synthetic_grid.argtypes = [vp, i32, vp, i32, vp, i32, vp, vp, vp, vp]
    lib.pp_synthetic_dataset.argtypes = [i64, vp, vp, i64, C.c_uint64, vp]
    lib.pp_slice_cost_host.argtypes = [C.POINTER(GridDesc), C.POINTER(ModelDesc), vp, i64, i64, vp, vp]
    lib.pp_calibrate_fp64.argtypes = [C.c_int, C.POINTER(dbl)]
    lib.pp_op_costs.argtypes = [vp, vp, i64, C.POINTER(GridDesc), C.POINTER(ModelDesc), vp, vp, vp]
    lib.pp_format_plan.argtypes = [vp, vp, i32, i32, vp, C.POINTER(ModelDesc), i64, i32, i64, C.c_char_p, i64, vp]
    lib.pp_emit_plans.argtypes = [vp, vp, vp, vp, vp, i32, i32, vp, C.c_double, i32, vp, vp, vp, vp, vp, vp, vp, vp]
    lib.pp_select_recomputation.argtypes = [vp, vp, vp, i32, C.POINTER(GridDesc), C.POINTER(ModelDesc), i32, vp,
                                            vp, vp, vp, vp, vp]
    lib.pp_select_recomputation_device.argtypes = [vp, vp, vp, vp, i32, vp, vp, C.POINTER(GridDesc),
                                                   C.POINTER(ModelDesc), i32, vp, i64, vp, vp, vp, vp, vp, vp]
    lib.pp_plan_op_costs_device.argtypes = [vp, vp, vp, vp, i32, vp, vp, C.POINTER(GridDesc),
                                            C.POINTER(ModelDesc), i64, vp, vp, vp, vp]
    lib.pp_load_records.argtypes = [vp, vp, i64, i64, vp, i64, vp, vp, vp, vp]
    lib.pp_load_records_device.argtypes = [vp, vp, i64, i64, vp, i64, vp, vp, vp, vp]
    lib.pp_draw_minibatches.argtypes = [vp, vp, i64, i64, vp, vp]
    lib.pp_draw_minibatches_device.argtypes = [vp, vp, i64, i64, vp, vp]
    lib.pp_padding_report.argtypes = [vp, vp, i64, vp, i32, C.POINTER(GridDesc), C.POINTER(ModelDesc), i64, dbl,
                                      i32, i32, vp]
    lib.pp_order_search.argtypes = [vp, vp, vp, vp, vp, i32, i32, vp, i32, dbl, vp, vp, vp, vp, vp, vp]
    lib.pp_order_search_device.argtypes = [vp, vp, vp, vp, vp, vp, i32, i32, vp, i32, dbl, vp, vp, vp, vp,
                                           vp, vp]
    return lib


lib = _load()


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ------------------------------------------------------------ host objects
@dataclass
class Grid:
    """A ProfileGrid as flat arrays (cost_model.h:74-105 layout)."""
    mbs_axis: np.ndarray
    seq_axis: np.ndarray
    cells: np.ndarray  # (2, 3, n_mbs, n_seq, 3) float64

    def desc(self) -> GridDesc:
        self.mbs_axis = np.ascontiguousarray(self.mbs_axis, dtype=np.int64)
        self.seq_axis = np.ascontiguousarray(self.seq_axis, dtype=np.int64)
        self.cells = np.ascontiguousarray(self.cells, dtype=np.float64)
        return GridDesc(len(self.mbs_axis), len(self.seq_axis), _p(self.mbs_axis),
                        _p(self.seq_axis), _p(self.cells))


@dataclass
class Model:
    """ModelConfig (cost_model.h:113-127) + the Recompute passed to make_slice_cost."""
    encoder_layers: np.ndarray
    decoder_layers: np.ndarray
    is_encoder_decoder: bool = False
    recompute: int = 0

    @staticmethod
    def uniform(n_stages: int, layers_per_stage: int, encoder_decoder: bool, recompute: int = 0):
        """ModelConfig::uniform (cost_model.cpp:273-292)."""
        if n_stages < 1 or layers_per_stage < 1:
            raise InvalidArgument("stage and layer counts must be >= 1")
        enc = np.zeros(n_stages, np.int32)
        dec = np.full(n_stages, layers_per_stage, np.int32)
        if encoder_decoder:
            if n_stages == 1:
                enc[0] = layers_per_stage
            else:
                ne = (n_stages + 1) // 2
                enc[:ne] = layers_per_stage
                dec[:ne] = 0
        return Model(enc, dec, encoder_decoder, recompute)

    def desc(self) -> ModelDesc:
        self.encoder_layers = np.ascontiguousarray(self.encoder_layers, dtype=np.int32)
        self.decoder_layers = np.ascontiguousarray(self.decoder_layers, dtype=np.int32)
        return ModelDesc(len(self.encoder_layers), _p(self.encoder_layers), _p(self.decoder_layers),
                         int(self.is_encoder_decoder), int(self.recompute))


SYNTH_DEFAULTS = dict(alpha=0.4, beta=2e-4, gamma=0.02, full_mem_factor=0.2,
                      selective_mem_factor=0.6, full_tb_penalty=1.0, selective_tb_penalty=0.5)


def synthetic_grid(mbs_axis=(), seq_axis=(), tp_degree: int = 1, **params) -> Grid:
    """ProfileGrid::synthetic via the library's host implementation."""
    p = dict(SYNTH_DEFAULTS)
    p.update(params)
    par = np.array([p[k] for k in ("alpha", "beta", "gamma", "full_mem_factor",
                                   "selective_mem_factor", "full_tb_penalty",
                                   "selective_tb_penalty")], np.float64)
    ma = np.asarray(mbs_axis, np.int64)
    sa = np.asarray(seq_axis, np.int64)
    om = np.zeros(64, np.int64)
    os_ = np.zeros(64, np.int64)
    sizes = np.zeros(2, np.int32)
    cells = np.zeros(18 * 64 * 64, np.float64)
    rc = lib.pp_synthetic_grid(_p(par), tp_degree, _p(ma), len(ma), _p(sa), len(sa), _p(om), _p(os_),
                               _p(sizes), _p(cells))
    if rc != PP_OK:
        raise InvalidArgument("synthetic grid coefficients must be positive")
    nm, ns = int(sizes[0]), int(sizes[1])
    return Grid(om[:nm].copy(), os_[:ns].copy(), cells[:18 * nm * ns].reshape(2, 3, nm, ns, 3).copy())


LOGNORMAL, UNIFORM, MIXTURE = 0, 1, 2


def synthetic_dataset(n: int, max_seq_len: int, seed: int, input_dist=(LOGNORMAL, 5.0, 1.5, 1, 1, 0.8),
                      target_dist=None) -> np.ndarray:
    """load_dataset(DatasetSpec{synthetic}) — byte-identical to the reference generator."""
    out = np.zeros((n, 3), np.int64)
    ind = np.asarray(input_dist, np.float64)
    tgd = None if target_dist is None else np.asarray(target_dist, np.float64)
    rc = lib.pp_synthetic_dataset(n, _p(ind), _p(tgd), max_seq_len, seed, _p(out))
    if rc != PP_OK:
        raise InvalidArgument("invalid synthetic dataset spec")
    return out


def slice_cost_host(grid: Grid, model: Model, ordered: np.ndarray, begin: int, end: int):
    t = np.zeros(1)
    m = np.zeros(1)
    ordered = np.ascontiguousarray(ordered, np.int64)
    rc = lib.pp_slice_cost_host(C.byref(grid.desc()), C.byref(model.desc()), _p(ordered), begin, end,
                                _p(t), _p(m))
    if rc != PP_OK:
        raise InvalidArgument("slice cost failed")
    return float(t[0]), float(m[0])


def calibrate_fp64(device: int = 0) -> float:
    """Measured FP64 add rate of the device (adds/s), see calib.cu."""
    out = C.c_double(0.0)
    rc = lib.pp_calibrate_fp64(device, C.byref(out))
    if rc != PP_OK:
        _raise_status(rc, -1, "fp64 calibration failed")
    return out.value


def assign_replicas(times, replica_count: int):
    """dp_partition's tail (microbatch.cpp:337-348) on the planned times:
    (replica per micro-batch, max_replica_load)."""
    t = np.ascontiguousarray(times, np.float64)
    rep = np.zeros(max(len(t), 1), np.int32)
    ml = np.zeros(1)
    rc = lib.pp_assign_replicas(_p(t), len(t), replica_count, _p(rep), _p(ml))
    if rc != PP_OK:
        raise InvalidArgument("replica assignment needs at least one micro-batch and replica_count >= 1")
    return rep[:len(t)].copy(), float(ml[0])


def eval_objective(times, stage_count: int, replica_count: int) -> float:
    t = np.ascontiguousarray(times, np.float64)
    out = np.zeros(1)
    rc = lib.pp_eval_objective(_p(t), len(t), stage_count, replica_count, _p(out))
    if rc != PP_OK:
        raise InvalidArgument("objective needs at least one micro-batch and counts >= 1")
    return float(out[0])


@dataclass
class Plan:
    """One mini-batch's plan: what dp_partition returns, in flat form."""
    status: int
    splits: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    mb_times: np.ndarray = field(default_factory=lambda: np.zeros(0))
    t_max_used: float = math.nan
    objective: float = math.nan
    err_sample_id: int = -1
    ordered: np.ndarray | None = None
    # dp_partition's tail (microbatch.cpp:337-348): replica_assignment and
    # max_replica_load (pp_assign_replicas)
    replica: np.ndarray | None = None
    max_load: float = math.nan
    # the candidate loop's counters: |unique candidates| and the candidates
    # the reference's loop visits before its break (pp_stats)
    n_candidates: int = -1
    n_evaluated: int = -1


def _raise_status(status: int, err_id: int, msg: str = ""):
    if status == PP_ERR_INFEASIBLE_SAMPLE:
        raise InfeasibleError(f"sample {err_id} does not fit the per-micro-batch memory cap alone",
                              err_id, -1)
    if status == PP_ERR_INFEASIBLE:
        raise InfeasibleError("no feasible partition under the memory cap", -1, -1)
    if status == PP_ERR_INVALID:
        raise InvalidArgument(msg or "invalid argument")
    if status == PP_ERR_NO_DEVICE:
        raise NoDeviceError("no CUDA device: the B200 planner has no CPU fallback")
    raise PlannerError(f"planner error {status}: {msg}")


class Planner:
    """A pp_ctx: one CUDA stream + scratch on one device."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        rc = lib.pp_ctx_create(device, C.byref(h))
        if rc != PP_OK:
            _raise_status(rc, -1, "cannot create context")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib.pp_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _err(self) -> str:
        return (lib.pp_ctx_last_error(self._h) or b"").decode()

    def set_tuning(self, first_wave: int = 1, max_wave: int = 16, streams: int = 1, coop_min_n: int = 0,
                   slice_reuse: bool = True, band_trunc: bool = True, compact_band: bool = False,
                   host_chunks: int = 0, dp_pricing: bool = False, slice_table: bool = True,
                   bin_intervals: bool = True):
        t = Tuning(first_wave, max_wave, streams, coop_min_n, 0 if slice_reuse else 1, 0 if band_trunc else 1,
                   1 if compact_band else 0, host_chunks, 1 if dp_pricing else 0,
                   0 if slice_table else 1, 0 if bin_intervals else 1)
        rc = lib.pp_ctx_set_tuning(self._h, C.byref(t))
        if rc != PP_OK:
            _raise_status(rc, -1, self._err())

    def set_stream(self, stream_ptr: int):
        lib.pp_ctx_set_stream(self._h, C.c_void_p(stream_ptr))

    def stats(self) -> dict:
        s = Stats()
        lib.pp_ctx_get_stats(self._h, C.byref(s))
        return s.as_dict()

    def order_samples(self, samples: np.ndarray, seg_offsets=None) -> np.ndarray:
        samples = np.ascontiguousarray(samples, np.int64).reshape(-1, 3)
        off = np.asarray([0, len(samples)] if seg_offsets is None else seg_offsets, np.int64)
        out = np.empty_like(samples)
        rc = lib.pp_order_samples(self._h, _p(samples), _p(off), len(off) - 1, _p(out))
        if rc != PP_OK:
            _raise_status(rc, -1, self._err())
        return out

    @staticmethod
    def plan_buffers(n_samples: int, n_seg: int, alloc=np.zeros, order_only: bool = False) -> dict:
        """Output arrays for plan_batch; pass e.g. a pinned-memory allocator
        (bench.py) so the device->host copies run at full PCIe rate.
        order_only: return the ordering as per-segment sample indices
        (`order`, 4 B per sample) instead of the ordered sample records."""
        if order_only:
            o = dict(ordered=None, order=alloc(max(n_samples, 1), np.int32))
        else:
            o = dict(ordered=alloc((max(n_samples, 1), 3), np.int64), order=None)
        return dict(**o,
                    splits=alloc(max(n_samples, 1), np.int32), mb_times=alloc(max(n_samples, 1), np.float64),
                    count=alloc(n_seg, np.int32), t_max_used=alloc(n_seg, np.float64),
                    objective=alloc(n_seg, np.float64), status=alloc(n_seg, np.int32),
                    err_sample_id=alloc(n_seg, np.int64))

    def plan_batch(self, samples: np.ndarray, seg_offsets, grid: Grid, model: Model, stage_count: int,
                   replica_count: int = 1, mem_cap: float = math.inf, t_max_interval: float = 5.0,
                   presorted: bool = False, out: dict | None = None) -> dict:
        """pp_plan_grid over independent mini-batches; returns flat arrays
        (written into `out` when given, see plan_buffers)."""
        samples = np.ascontiguousarray(samples, np.int64).reshape(-1, 3)
        off = np.ascontiguousarray(seg_offsets, np.int64)
        S = len(off) - 1
        n = len(samples)
        res = dict(out) if out is not None else self.plan_buffers(n, S)
        out = PlanOut(*(_p(res.get(k)) for k in ("ordered", "splits", "mb_times", "count", "t_max_used",
                                                "objective", "status", "err_sample_id", "order")))
        g, m = grid.desc(), model.desc()
        o = DpOptions(stage_count, replica_count, mem_cap, t_max_interval)
        rc = lib.pp_plan_grid(self._h, _p(samples), _p(off), S, int(presorted), C.byref(g), C.byref(m),
                              C.byref(o), C.byref(out))
        if rc != PP_OK:
            _raise_status(rc, -1, self._err())
        res["seg_offsets"] = off
        return res

    def plan_batch_device(self, d_samples, d_seg_offsets, h_seg_offsets, d_out: dict, grid: Grid,
                          model: Model, stage_count: int, replica_count: int = 1,
                          mem_cap: float = math.inf, t_max_interval: float = 5.0,
                          presorted: bool = False) -> None:
        """pp_plan_grid_device: inputs and outputs are device tensors (torch),
        already resident in HBM.  d_out maps the pp_plan_out field names to
        device tensors."""
        h_off = np.ascontiguousarray(h_seg_offsets, np.int64)
        S = len(h_off) - 1
        out = PlanOut(*(C.c_void_p(d_out[k].data_ptr()) if d_out.get(k) is not None else None
                        for k in ("ordered", "splits", "mb_times", "count", "t_max_used", "objective",
                                  "status", "err_sample_id", "order")))
        g, m = grid.desc(), model.desc()
        o = DpOptions(stage_count, replica_count, mem_cap, t_max_interval)
        rc = lib.pp_plan_grid_device(self._h, C.c_void_p(d_samples.data_ptr()),
                                     C.c_void_p(d_seg_offsets.data_ptr()), _p(h_off), S, int(presorted),
                                     C.byref(g), C.byref(m), C.byref(o), C.byref(out))
        if rc != PP_OK:
            _raise_status(rc, -1, self._err())

    def pack_slots_device(self, d_out: dict, d_seg_offsets, n_seg: int, n_max: int, d_slots,
                          with_order: bool = True) -> None:
        """pp_pack_plan_slots: the device plan outputs (pp_plan_out field
        names -> torch tensors) -> fixed-size int64 slots (d_slots, a torch
        tensor of n_seg x slot words), on the planner's stream."""
        vp = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
        order = d_out.get("order") if with_order else None
        if with_order and order is None:
            raise InvalidArgument("with_order needs the 'order' output")
        rc = lib.pp_pack_plan_slots(self._h, vp(d_out["count"]), vp(d_out["status"]), vp(d_out["t_max_used"]),
                                    vp(d_out["objective"]), vp(d_out["splits"]), vp(order), vp(d_seg_offsets),
                                    n_seg, n_max, vp(d_slots))
        if rc != PP_OK:
            _raise_status(rc, -1, self._err())

    def plan(self, samples: np.ndarray, grid: Grid, model: Model, stage_count: int,
             replica_count: int = 1, mem_cap: float = math.inf, t_max_interval: float = 5.0,
             presorted: bool = False) -> Plan:
        """order_samples(Sort) + make_slice_cost + dp_partition for one mini-batch;
        raises like the reference does."""
        r = self.plan_batch(samples, [0, len(samples)], grid, model, stage_count, replica_count,
                            mem_cap, t_max_interval, presorted)
        st = int(r["status"][0])
        if st != PP_OK:
            _raise_status(st, int(r["err_sample_id"][0]), self._err())
        m = int(r["count"][0])
        times = r["mb_times"][:m].copy()
        rep, ml = assign_replicas(times, replica_count)
        st_ = self.stats()
        return Plan(st, r["splits"][:m].copy(), times, float(r["t_max_used"][0]),
                    float(r["objective"][0]), -1, r["ordered"], rep, ml,
                    int(st_["candidates_generated"]), int(st_["candidates_ref_evaluated"]))

    def plan_tables(self, T: np.ndarray, M: np.ndarray, n: int, stage_count: int,
                    replica_count: int = 1, mem_cap: float = math.inf,
                    t_max_interval: float = 5.0) -> Plan:
        """dp_partition with a generic SliceCostFn given as triangular tables."""
        T = np.ascontiguousarray(T, np.float64)
        M = np.ascontiguousarray(M, np.float64)
        splits = np.zeros(max(n, 1), np.int32)
        times = np.zeros(max(n, 1))
        cnt = np.zeros(1, np.int32)
        tm = np.zeros(1)
        ob = np.zeros(1)
        err = np.full(1, -1, np.int64)
        o = DpOptions(stage_count, replica_count, mem_cap, t_max_interval)
        rc = lib.pp_plan_tables(self._h, _p(T), _p(M), n, C.byref(o), _p(splits), _p(times), _p(cnt),
                                _p(tm), _p(ob), _p(err))
        if rc != PP_OK:
            _raise_status(rc, int(err[0]), self._err())
        m = int(cnt[0])
        rep, ml = assign_replicas(times[:m], replica_count)
        st_ = self.stats()
        return Plan(PP_OK, splits[:m].copy(), times[:m].copy(), float(tm[0]), float(ob[0]), -1, None, rep, ml,
                    int(st_["candidates_generated"]), int(st_["candidates_ref_evaluated"]))

    def op_costs(self, shapes, grid: Grid, model: Model):
        """OpCostTable::from_shapes: (t_f, t_b, act_mem), each (n, n_stages);
        shapes is an (n, 3) int64 array of (mbs, input_len, target_len)."""
        sh = np.ascontiguousarray(shapes, np.int64).reshape(-1, 3)
        n, C_ = len(sh), len(model.encoder_layers)
        tf, tb, act = (np.zeros((n, C_)) for _ in range(3))
        rc = lib.pp_op_costs(self._h, _p(sh), n, C.byref(grid.desc()), C.byref(model.desc()), _p(tf),
                             _p(tb), _p(act))
        if rc != PP_OK:
            _raise_status(rc, -1, self._err())
        return tf, tb, act

    def select_recomputation(self, shapes, mb_offset, grid: Grid, model: Model, strategies=(0, 1, 2),
                             limits=None) -> dict:
        """select_recomputation per partition (rows mb_offset[s]..[s+1] of
        shapes): {"strategy": (S,) Recompute or -1, "violating_stage": (S,),
        "t_f"/"t_b"/"act_mem": (rows, n_stages) of the chosen strategy}."""
        sh = np.ascontiguousarray(shapes, np.int64).reshape(-1, 3)
        off = np.ascontiguousarray(mb_offset, np.int64)
        S, C_ = len(off) - 1, len(model.encoder_layers)
        lim = np.ascontiguousarray(limits, np.float64)
        mask = sum(1 << int(r) for r in strategies)
        tf, tb, act = (np.zeros((max(len(sh), 1), C_)) for _ in range(3))
        st, vs = np.zeros(S, np.int32), np.zeros(S, np.int32)
        rc = lib.pp_select_recomputation(self._h, _p(sh), _p(off), S, C.byref(grid.desc()), C.byref(model.desc()),
                                         mask, _p(lim), _p(tf), _p(tb), _p(act), _p(st), _p(vs))
        if rc != PP_OK:
            _raise_status(rc, -1, self._err())
        n = len(sh)
        return {"strategy": st, "violating_stage": vs, "t_f": tf[:n], "t_b": tb[:n], "act_mem": act[:n]}

    def select_recomputation_device(self, d_ordered, d_seg_offsets, h_seg_offsets, d_splits, d_count,
                                    grid: Grid, model: Model, limits, d_tf, d_tb, d_act, d_strategy,
                                    d_violating, strategies=(0, 1, 2)) -> np.ndarray:
        """select_recomputation for every plan already on the device; returns
        mb_offset (host); tables / strategy / violating stage into the d_* tensors."""
        h_off = np.ascontiguousarray(h_seg_offsets, np.int64)
        S = len(h_off) - 1
        mb_off = np.zeros(S + 1, np.int64)
        cap = d_tf.numel() // len(model.encoder_layers)
        lim = np.ascontiguousarray(limits, np.float64)
        mask = sum(1 << int(r) for r in strategies)
        rc = lib.pp_select_recomputation_device(
            self._h, C.c_void_p(d_ordered.data_ptr()), C.c_void_p(d_seg_offsets.data_ptr()), _p(h_off), S,
            C.c_void_p(d_splits.data_ptr()), C.c_void_p(d_count.data_ptr()), C.byref(grid.desc()),
            C.byref(model.desc()), mask, _p(lim), cap, _p(mb_off), C.c_void_p(d_tf.data_ptr()),
            C.c_void_p(d_tb.data_ptr()), C.c_void_p(d_act.data_ptr()), C.c_void_p(d_strategy.data_ptr()),
            C.c_void_p(d_violating.data_ptr()))
        if rc != PP_OK:
            _raise_status(rc, -1, self._err())
        return mb_off

    def emit_plans(self, t_f, t_b, act_mem, mb_offset, limits=None, order=None, comm_latency=0.0,
                   one_f_one_b=False) -> dict:
        """The chosen plan per table: {"instructions": list (table) of lists
        (stage) of (InstrKind, micro_batch) int32 arrays, "makespan",
        "bubble_ratio", "deadlock", "device_stats" (S, C, 5), "status"}."""
        tf = np.ascontiguousarray(t_f, np.float64)
        C_ = tf.shape[1]
        tb = np.ascontiguousarray(t_b, np.float64)
        ac = np.ascontiguousarray(act_mem, np.float64)
        off = np.ascontiguousarray(mb_offset, np.int64)
        S = len(off) - 1
        rows = int(off[-1])
        ins = np.zeros(max(rows, 1) * 10 * C_, np.int32)
        nins = np.zeros((S, C_), np.int32)
        ms, bub = np.zeros(S), np.zeros(S)
        dl, st = np.zeros(S, np.int32), np.zeros(S, np.int32)
        ds = np.zeros((S, C_, 5))
        lim = np.ascontiguousarray(limits if limits is not None else np.zeros(C_), np.float64)
        od = np.ascontiguousarray(order if order is not None else np.zeros(max(rows, 1)), np.int32)
        rc = lib.pp_emit_plans(self._h, _p(tf), _p(tb), _p(ac), _p(off), S, C_, _p(lim), comm_latency,
                               1 if one_f_one_b else 0, _p(od), _p(ins), _p(nins), _p(ms), _p(bub), _p(dl),
                               _p(ds), _p(st))
        if rc != PP_OK:
            _raise_status(rc, -1, self._err())
        lists = []
        for s in range(S):
            m = int(off[s + 1] - off[s])
            per = []
            for j in range(C_):
                a = ins[10 * C_ * off[s] + 10 * m * j: 10 * C_ * off[s] + 10 * m * j + nins[s, j]]
                per.append(np.stack([a & 15, a >> 4], 1).astype(np.int32))
            lists.append(per)
        return {"instructions": lists, "makespan": ms, "bubble_ratio": bub, "deadlock": dl, "device_stats": ds,
                "status": st}

    @staticmethod
    def format_plan(instructions, shapes, model: "Model", iteration=0, replica=0, hidden_dim=1024) -> str:
        """save_plan's text of one emitted plan: instructions = emit_plans(...)
        ["instructions"][s] (per stage (kind, micro_batch) rows)."""
        C_ = len(instructions)
        sh = np.ascontiguousarray(shapes, np.int64).reshape(-1, 3)
        M = len(sh)
        ins = np.zeros(max(M, 1) * 10 * C_, np.int32)
        nins = np.zeros(C_, np.int32)
        for j, a in enumerate(instructions):
            packed = (np.asarray(a)[:, 1] << 4) | np.asarray(a)[:, 0] if len(a) else np.zeros(0, np.int32)
            ins[10 * M * j:10 * M * j + len(packed)] = packed
            nins[j] = len(packed)
        n = np.zeros(1, np.int64)
        md = model.desc()
        buf = C.create_string_buffer(1 << 22)
        rc = lib.pp_format_plan(_p(ins), _p(nins), C_, M, _p(sh), C.byref(md), iteration, replica, hidden_dim, buf,
                                len(buf), _p(n))
        if rc != PP_OK:
            raise InvalidArgument("bad plan")
        return buf.value.decode()

    def plan_op_costs_device(self, d_ordered, d_seg_offsets, h_seg_offsets, d_splits, d_count,
                             grid: Grid, model: Model, d_tf, d_tb, d_act) -> np.ndarray:
        """Op-cost tables of every planned micro-batch (device tensors);
        returns mb_offset (host)."""
        h_off = np.ascontiguousarray(h_seg_offsets, np.int64)
        S = len(h_off) - 1
        mb_off = np.zeros(S + 1, np.int64)
        cap = d_tf.numel() // len(model.encoder_layers)
        rc = lib.pp_plan_op_costs_device(
            self._h, C.c_void_p(d_ordered.data_ptr()), C.c_void_p(d_seg_offsets.data_ptr()), _p(h_off), S,
            C.c_void_p(d_splits.data_ptr()), C.c_void_p(d_count.data_ptr()), C.byref(grid.desc()),
            C.byref(model.desc()), cap, _p(mb_off), C.c_void_p(d_tf.data_ptr()),
            C.c_void_p(d_tb.data_ptr()), C.c_void_p(d_act.data_ptr()))
        if rc != PP_OK:
            _raise_status(rc, -1, self._err())
        return mb_off

    def load_records(self, data: bytes, max_seq_len: int, capacity: int | None = None):
        """load_dataset over a record file's bytes on the device -> (n, 3)
        int64 samples.  Raises ParseError (line, byte) / InvalidArgument."""
        buf = np.frombuffer(data, np.uint8)
        cap = len(buf) // 2 + 1 if capacity is None else capacity
        out = np.zeros((cap, 3), np.int64)
        n, el, eb = (np.zeros(1, np.int64) for _ in range(3))
        ek = np.zeros(1, np.int32)
        rc = lib.pp_load_records(self._h, _p(buf) if len(buf) else None, len(buf), max_seq_len, _p(out), cap,
                                 _p(n), _p(el), _p(eb), _p(ek))
        if rc == PP_ERR_PARSE:
            raise ParseError(self._err(), int(el[0]), int(eb[0]), int(ek[0]))
        if rc != PP_OK:
            _raise_status(rc, -1, self._err())
        return out[:int(n[0])].copy()

    def load_records_device(self, d_bytes, n_bytes: int, max_seq_len: int, d_out) -> int:
        n, el, eb = (np.zeros(1, np.int64) for _ in range(3))
        ek = np.zeros(1, np.int32)
        rc = lib.pp_load_records_device(self._h, C.c_void_p(d_bytes.data_ptr()), n_bytes, max_seq_len,
                                        C.c_void_p(d_out.data_ptr()), d_out.shape[0], _p(n), _p(el), _p(eb),
                                        _p(ek))
        if rc == PP_ERR_PARSE:
            raise ParseError(self._err(), int(el[0]), int(eb[0]), int(ek[0]))
        if rc != PP_OK:
            _raise_status(rc, -1, self._err())
        return int(n[0])

    def draw_minibatches(self, samples, token_budget: int) -> np.ndarray:
        """run_plan's draw_minibatch loop -> seg_offsets (n_seg + 1)."""
        s = np.ascontiguousarray(samples, np.int64).reshape(-1, 3)
        off = np.zeros(len(s) + 1, np.int64)
        m = np.zeros(1, np.int64)
        rc = lib.pp_draw_minibatches(self._h, _p(s) if len(s) else None, len(s), token_budget, _p(off), _p(m))
        if rc != PP_OK:
            _raise_status(rc, -1, self._err())
        return off[:int(m[0]) + 1].copy()

    def draw_minibatches_device(self, d_samples, n: int, token_budget: int, d_offsets) -> int:
        m = np.zeros(1, np.int64)
        rc = lib.pp_draw_minibatches_device(self._h, C.c_void_p(d_samples.data_ptr()), n, token_budget,
                                            C.c_void_p(d_offsets.data_ptr()), _p(m))
        if rc != PP_OK:
            _raise_status(rc, -1, self._err())
        return int(m[0])

    def padding_report(self, samples, max_seq_lens, grid: "Grid", model: "Model", token_budget: int = 65536,
                       t_max_interval: float = 5.0, max_iterations: int = 0, recompute: int = 0) -> np.ndarray:
        """padding_vs_packing_report on the device -> structured rows (3 per max_seq_len)."""
        s = np.ascontiguousarray(samples, np.int64).reshape(-1, 3)
        lens = np.ascontiguousarray(max_seq_lens, np.int64)
        rows = np.zeros(3 * len(lens), PADDING_ROW)
        rc = lib.pp_padding_report(self._h, _p(s) if len(s) else None, len(s), _p(lens), len(lens),
                                   C.byref(grid.desc()), C.byref(model.desc()), token_budget, t_max_interval,
                                   max_iterations, recompute, rows.ctypes.data)
        if rc != PP_OK:
            _raise_status(rc, -1, self._err())
        return rows

    def order_search(self, t_f, t_b, act_mem, mb_offset, limits, n_clusters: int = 3,
                     comm_latency: float = 0.0) -> dict:
        """order_microbatches with the planner's simulate(plan_communication(...))
        evaluator over every op-cost table [mb_offset[s], mb_offset[s+1]) of the
        (rows, n_stages) arrays.  Returns a dict of per-table arrays: order
        (rows), makespan, bubble_ratio, deadlock, device_stats (n_seg, C, 5),
        status."""
        tf = np.ascontiguousarray(t_f, np.float64)
        tb = np.ascontiguousarray(t_b, np.float64)
        ac = np.ascontiguousarray(act_mem, np.float64)
        off = np.ascontiguousarray(mb_offset, np.int64)
        lim = np.ascontiguousarray(limits, np.float64)
        S, C_ = len(off) - 1, tf.shape[1]
        out = {"order": np.full(len(tf), -1, np.int32), "makespan": np.zeros(S), "bubble_ratio": np.zeros(S),
               "deadlock": np.zeros(S, np.int32), "device_stats": np.zeros((S, C_, 5)),
               "status": np.zeros(S, np.int32)}
        rc = lib.pp_order_search(self._h, _p(tf), _p(tb), _p(ac), _p(off), S, C_, _p(lim), n_clusters,
                                 float(comm_latency), _p(out["order"]), _p(out["makespan"]),
                                 _p(out["bubble_ratio"]), _p(out["deadlock"]), _p(out["device_stats"]),
                                 _p(out["status"]))
        if rc != PP_OK:
            _raise_status(rc, -1, self._err())
        return out

    def order_search_device(self, d_tf, d_tb, d_act, d_mb_offset, h_mb_offset, limits, d_out: dict,
                            n_clusters: int = 3, comm_latency: float = 0.0) -> None:
        """Device-resident variant (torch tensors); d_out holds order, makespan,
        bubble_ratio, deadlock, device_stats (may be None), status."""
        off = np.ascontiguousarray(h_mb_offset, np.int64)
        lim = np.ascontiguousarray(limits, np.float64)
        S, C_ = len(off) - 1, len(lim)
        ptr = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
        rc = lib.pp_order_search_device(
            self._h, ptr(d_tf), ptr(d_tb), ptr(d_act), ptr(d_mb_offset), _p(off), S, C_, _p(lim), n_clusters,
            float(comm_latency), ptr(d_out["order"]), ptr(d_out["makespan"]), ptr(d_out.get("bubble_ratio")),
            ptr(d_out.get("deadlock")), ptr(d_out.get("device_stats")), ptr(d_out["status"]))
        if rc != PP_OK:
            _raise_status(rc, -1, self._err())

    def candidate_range(self, samples, seg_offsets, grid: Grid, model: Model,
                        mem_cap: float = math.inf, presorted: bool = False):
        samples = np.ascontiguousarray(samples, np.int64).reshape(-1, 3)
        off = np.ascontiguousarray(seg_offsets, np.int64)
        S = len(off) - 1
        lo = np.zeros(S)
        hi = np.zeros(S)
        rc = lib.pp_candidate_range(self._h, _p(samples), _p(off), S, int(presorted),
                                    C.byref(grid.desc()), C.byref(model.desc()), mem_cap, _p(lo),
                                    _p(hi))
        if rc != PP_OK:
            _raise_status(rc, -1, self._err())
        return lo, hi
