"""ctypes binding of libparo.so (include/paro.h).  Argument marshalling only:
every step of the PaRO sync + update path runs in the library's kernels.

The functions keep the C names (paro_init, paro_plan, paro_step, ...); the
small `Context` / `Plan` classes below only hold handles and turn status
codes into exceptions.  There is no CPU fallback: if the shared library is
missing this module raises at import time.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libparo.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")

_lib = C.CDLL(LIB_PATH)

# ---------------------------------------------------------------- constants
PARO_OK, PARO_ERR_INVALID, PARO_ERR_OOM, PARO_ERR_CUDA, PARO_ERR_NCCL, PARO_ERR_STATE, PARO_ERR_TIMEOUT = range(7)
TOPO = {"ho": 0, "two_step": 1, "flat": 2, "direct": 3, "nccl": 4, "h_ring": 5, "oneshot": 6}
STATE = {"P": 0, "G": 1, "OS": 2}


class ParoError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"[paro status {status}] {msg}")
        self.status = status


# ---------------------------------------------------------------- structs
class paro_uid_t(C.Structure):
    _fields_ = [("bytes", C.c_char * 128)]


class paro_opt_state_t(C.Structure):
    _fields_ = [("master", C.c_void_p), ("m", C.c_void_p), ("v", C.c_void_p)]


class paro_opts_t(C.Structure):
    _fields_ = [("bucket_elems", C.c_int64), ("topology", C.c_int), ("beta1", C.c_float),
                ("beta2", C.c_float), ("eps", C.c_float), ("weight_decay", C.c_float),
                ("loss_scale", C.c_float), ("comm_ctas", C.c_int), ("pipeline_depth", C.c_int),
                ("pull_transport", C.c_int), ("adam_impl", C.c_int), ("comm_impl", C.c_int),
                ("inter_gbps", C.c_float), ("clip_norm", C.c_float), ("skip_nonfinite", C.c_int),
                ("fuse_gather", C.c_int), ("copy_engine", C.c_int), ("gather_windows", C.c_int), ("grad_accum", C.c_int),
                ("stream", C.c_void_p), ("frozen", C.c_int), ("grad_slots", C.c_int),
                ("fuse_allreduce", C.c_int), ("adam_smem_kb", C.c_int), ("wire_dtype", C.c_int),
                ("predivide", C.c_int), ("bucket_groups", C.POINTER(C.c_int64)), ("n_bucket_groups", C.c_int)]


class paro_plan_info_t(C.Structure):
    _fields_ = [("psi", C.c_int64), ("psi_pad", C.c_int64), ("bucket_elems", C.c_int64),
                ("n_buckets", C.c_int64), ("p_numel", C.c_int64), ("g_numel", C.c_int64),
                ("os_numel", C.c_int64), ("mem_p_bytes", C.c_int64), ("mem_g_bytes", C.c_int64),
                ("mem_os_bytes", C.c_int64), ("workspace_bytes", C.c_int64),
                ("step_send_bytes_intra", C.c_int64), ("step_send_bytes_inter", C.c_int64),
                ("n_rounds", C.c_int32), ("n_comm_launches", C.c_int32),
                ("accum_send_bytes_intra", C.c_int64), ("accum_send_bytes_inter", C.c_int64),
                ("accum_step_send_bytes_intra", C.c_int64), ("accum_step_send_bytes_inter", C.c_int64),
                ("grad_buffer_bytes", C.c_int64)]


class paro_step_stats_t(C.Structure):
    _fields_ = [("grad_norm", C.c_double), ("nonfinite", C.c_int32), ("sent_intra", C.c_int64),
                ("sent_inter", C.c_int64), ("kernel_launches", C.c_int32), ("moved_intra", C.c_int64),
                ("moved_inter", C.c_int64)]


class paro_profile_t(C.Structure):
    _fields_ = [("adam_ms", C.c_double), ("comm_ms", C.c_double), ("adam_launches", C.c_int64),
                ("comm_launches", C.c_int64), ("adam_elems", C.c_int64), ("comm_bytes", C.c_int64),
                ("steps", C.c_int64), ("kernel_launches", C.c_int64), ("traced_launches", C.c_int64),
                ("traced_barrier_ms", C.c_double), ("traced_work_ms", C.c_double), ("traced_final_ms", C.c_double),
                ("adam_hbm_bytes", C.c_int64), ("comm_hbm_bytes", C.c_int64),
                ("adam_variant", C.c_int32), ("adam_stages", C.c_int32)]

ADAM_VARIANTS = {-1: None, 0: "adam_kernel", 1: "adam_tma_kernel<false,512>", 2: "adam_tma_kernel<true,512>",
                 3: "adam_tma_kernel<true,256>", 4: "adam_tma_kernel<false,256>", 5: "adam_tma_ws_kernel<512>",
                 6: "adam_tma_ws_kernel<256>"}


class paro_advise_in_t(C.Structure):
    _fields_ = [("n_gpus", C.c_int), ("group_size", C.c_int), ("psi", C.c_int64), ("psi_trainable", C.c_int64),
                ("accum_steps", C.c_int), ("peft", C.c_int), ("mem_budget_bytes", C.c_double),
                ("bw_intra_gbs", C.c_double), ("bw_inter_gbs", C.c_double)]


class paro_advice_t(C.Structure):
    _fields_ = [("code", C.c_char * 4), ("recommended", C.c_int32), ("fits", C.c_int32), ("mem_bytes", C.c_int64),
                ("intra_bytes", C.c_int64), ("inter_bytes", C.c_int64), ("t_comm_s", C.c_double)]


_vp = C.c_void_p
_i64 = C.c_int64
_st = C.c_int


def _sig(name, restype, *argtypes):
    f = getattr(_lib, name)
    f.restype = restype
    f.argtypes = list(argtypes)
    return f


paro_opts_default = _sig("paro_opts_default", None, C.POINTER(paro_opts_t))
paro_get_unique_id = _sig("paro_get_unique_id", _st, C.POINTER(paro_uid_t))
paro_init = _sig("paro_init", _st, C.c_int, C.c_int, C.c_int, C.POINTER(paro_uid_t), C.c_int, C.POINTER(_vp))
paro_init_emulated = _sig("paro_init_emulated", _st, C.c_int, C.c_int, C.c_int, C.POINTER(_vp))
paro_init_planner = _sig("paro_init_planner", _st, C.c_int, C.c_int, C.POINTER(_vp))
paro_finalize = _sig("paro_finalize", _st, _vp)
paro_plan = _sig("paro_plan", _st, _vp, C.c_char_p, C.POINTER(_i64), C.c_int, C.POINTER(paro_opts_t),
                 C.POINTER(_vp))
paro_plan_masked = _sig("paro_plan_masked", _st, _vp, C.c_char_p, C.POINTER(_i64), C.POINTER(C.c_uint8), C.c_int,
                        C.POINTER(paro_opts_t), C.POINTER(_vp), C.POINTER(_vp))
paro_plan_info = _sig("paro_plan_info", _st, _vp, C.POINTER(paro_plan_info_t))
paro_shard_range = _sig("paro_shard_range", _st, _vp, C.c_int, C.c_int, _i64, C.POINTER(_i64), C.POINTER(_i64))
paro_bucket_range = _sig("paro_bucket_range", _st, _vp, _i64, C.POINTER(_i64), C.POINTER(_i64))
paro_rank_send_bytes = _sig("paro_rank_send_bytes", _st, _vp, C.c_int, C.POINTER(_i64), C.POINTER(_i64))
paro_rank_accum_send_bytes = _sig("paro_rank_accum_send_bytes", _st, _vp, C.c_int, C.POINTER(_i64),
                                  C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64))
paro_gather_window = _sig("paro_gather_window", _st, _vp, C.c_int, _i64, C.c_int, _vp, C.POINTER(_vp))
paro_rank_gather_send_bytes = _sig("paro_rank_gather_send_bytes", _st, _vp, C.c_int, C.POINTER(_i64),
                                   C.POINTER(_i64))
paro_bucket_gather_send_bytes = _sig("paro_bucket_gather_send_bytes", _st, _vp, C.c_int, _i64, C.POINTER(_i64),
                                     C.POINTER(_i64))
paro_buffer = _sig("paro_buffer", _st, _vp, C.c_int, C.c_int, C.POINTER(_vp))
paro_opt_state_init = _sig("paro_opt_state_init", _st, _vp, C.c_int, _vp, C.POINTER(paro_opt_state_t))
paro_opt_state_init_synth = _sig("paro_opt_state_init_synth", _st, _vp, C.c_int, C.c_uint64,
                                 C.POINTER(paro_opt_state_t))
paro_synth_grads = _sig("paro_synth_grads", _st, _vp, C.c_int, C.c_uint64, _i64)
paro_step = _sig("paro_step", _st, _vp, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(paro_opt_state_t),
                 C.c_float, _i64)
PRODUCER = C.CFUNCTYPE(None, C.c_void_p, C.c_int, _i64, _i64, _i64, C.c_void_p, C.c_void_p)
paro_step_streamed = _sig("paro_step_streamed", _st, _vp, PRODUCER, C.c_void_p, C.c_uint64, _i64, C.POINTER(_vp),
                          C.POINTER(paro_opt_state_t), C.c_float, _i64)
paro_accumulate = _sig("paro_accumulate", _st, _vp, C.POINTER(_vp))
CONSUMER = C.CFUNCTYPE(None, C.c_void_p, C.c_int, _i64, _i64, _i64, C.c_void_p, C.c_void_p)
paro_set_param_consumer = _sig("paro_set_param_consumer", _st, _vp, CONSUMER, C.c_void_p)
paro_step_stats = _sig("paro_step_stats", _st, _vp, C.POINTER(paro_step_stats_t))
paro_plan_destroy = _sig("paro_plan_destroy", _st, _vp)
paro_collective = _sig("paro_collective", _st, _vp, C.c_int)
paro_profile_start = _sig("paro_profile_start", _st, _vp, C.c_int)
paro_profile_stop = _sig("paro_profile_stop", _st, _vp, C.POINTER(paro_profile_t))
paro_table1_column = _sig("paro_table1_column", C.c_int, _i64, _i64, C.c_int)
paro_advise = _sig("paro_advise", _st, C.POINTER(paro_advise_in_t), C.POINTER(paro_advice_t), C.c_int,
                   C.POINTER(C.c_int))
paro_last_error = _sig("paro_last_error", C.c_char_p)
paro_version = _sig("paro_version", C.c_char_p)

EXPORTED = ["paro_opts_default", "paro_get_unique_id", "paro_init", "paro_init_emulated",
            "paro_init_planner", "paro_finalize", "paro_plan", "paro_plan_info", "paro_shard_range",
            "paro_bucket_range", "paro_rank_send_bytes", "paro_buffer", "paro_opt_state_init",
            "paro_opt_state_init_synth", "paro_synth_grads", "paro_step", "paro_step_stats",
            "paro_plan_destroy", "paro_last_error", "paro_version", "paro_profile_start",
            "paro_profile_stop", "paro_collective", "paro_accumulate",
            "paro_rank_accum_send_bytes", "paro_gather_window", "paro_rank_gather_send_bytes",
            "paro_table1_column", "paro_advise", "paro_plan_masked", "paro_step_streamed",
            "paro_bucket_gather_send_bytes", "paro_set_param_consumer"]


def check(status):
    if status != PARO_OK:
        raise ParoError(status, paro_last_error().decode())
    return status


# ---------------------------------------------------------------- helpers
def make_opts(bucket_elems=1 << 26, topology="ho", beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.0,
              loss_scale=1.0, comm_ctas=0, pipeline_depth=2, stream=None, transport="pull", adam_impl="auto",
              comm_impl="tma_store", inter_gbps=0.0, grad_accum=False, clip_norm=0.0, skip_nonfinite=False, gather_windows=0,
              fuse_gather="auto", copy_engine=False, frozen=False, grad_slots=0, fuse_allreduce=True,
              adam_smem_kb=0, wire_dtype="bf16", predivide=True, bucket_groups=None):
    o = paro_opts_t()
    paro_opts_default(C.byref(o))
    o.bucket_elems = int(bucket_elems)
    o.topology = TOPO[topology] if isinstance(topology, str) else int(topology)
    o.beta1, o.beta2, o.eps = beta1, beta2, eps
    o.weight_decay, o.loss_scale = weight_decay, loss_scale
    o.comm_ctas, o.pipeline_depth = int(comm_ctas), int(pipeline_depth)
    o.pull_transport = {"push": 0, "pull": 1}[transport]
    o.adam_impl = {"auto": 0, "lsu": 1, "tma_store": 2, "tma": 3, "tma_ws": 4}[adam_impl]
    o.comm_impl = {"tma": 0, "lsu": 1, "tma_store": 2}[comm_impl]
    o.inter_gbps = float(inter_gbps)
    o.grad_accum = 1 if grad_accum else 0
    o.clip_norm = float(clip_norm)
    o.skip_nonfinite = 1 if skip_nonfinite else 0
    o.gather_windows = int(gather_windows)
    o.fuse_gather = {"auto": 1, "always": 2, "never": 0, True: 2, False: 0}[fuse_gather]
    o.copy_engine = {False: 0, True: 1, "gathers": 1, "all": 2, "tails": 3, 0: 0, 1: 1, 2: 2, 3: 3}[copy_engine]
    o.stream = stream
    o.frozen = 1 if frozen else 0
    o.grad_slots = int(grad_slots)
    o.fuse_allreduce = 1 if fuse_allreduce else 0
    o.adam_smem_kb = int(adam_smem_kb)
    o.wire_dtype = {"bf16": 0, "fp32": 1, 0: 0, 1: 1}[wire_dtype]
    o.predivide = 1 if predivide else 0
    if bucket_groups is not None:
        arr = (_i64 * max(1, len(bucket_groups)))(*[int(x) for x in bucket_groups])
        o._groups_keep = arr            # the library reads it during paro_plan only
        o.bucket_groups = C.cast(arr, C.POINTER(C.c_int64))
        o.n_bucket_groups = len(bucket_groups)
    return o


def advise(n_gpus, group_size, psi, psi_trainable, accum_steps, mem_budget_bytes, bw_intra_gbs, bw_inter_gbs,
           peft=False):
    """paro_advise: the 14 strategies ranked for one training task (list of dicts, best first)."""
    a = paro_advise_in_t(int(n_gpus), int(group_size), int(psi), int(psi_trainable), int(accum_steps),
                         1 if peft else 0, float(mem_budget_bytes), float(bw_intra_gbs), float(bw_inter_gbs))
    out = (paro_advice_t * 14)()
    n = C.c_int()
    check(paro_advise(C.byref(a), out, 14, C.byref(n)))
    rows = []
    for x in out[:n.value]:
        rows.append({"code": x.code.decode(), "recommended": bool(x.recommended), "fits": bool(x.fits),
                     "mem_bytes": x.mem_bytes, "intra_bytes": x.intra_bytes, "inter_bytes": x.inter_bytes,
                     "t_s": x.t_comm_s})
    return rows


def unique_id():
    u = paro_uid_t()
    check(paro_get_unique_id(C.byref(u)))
    return C.string_at(C.addressof(u), 128)   # raw 128 bytes (the id contains NULs)


class Context:
    """paro_init (real rank), paro_init_emulated (all ranks, one device) or
    paro_init_planner (host only)."""

    def __init__(self, world_size, group_size, mode="planner", rank=0, device=0, uid=None):
        h = _vp()
        if mode == "planner":
            check(paro_init_planner(world_size, group_size, C.byref(h)))
        elif mode == "emulated":
            check(paro_init_emulated(world_size, group_size, device, C.byref(h)))
        elif mode == "real":
            u = paro_uid_t()
            assert uid is not None and len(uid) == 128, "uid must be the 128 raw bytes of unique_id()"
            C.memmove(C.addressof(u), bytes(uid), 128)
            check(paro_init(world_size, group_size, rank, C.byref(u), device, C.byref(h)))
        else:
            raise ValueError(mode)
        self.h, self.mode, self.N, self.M, self.rank = h, mode, world_size, group_size, rank

    def close(self):
        if self.h:
            paro_finalize(self.h)
            self.h = None


class Plan:
    @classmethod
    def masked(cls, ctx, strategy, param_sizes, trainable, **opts):
        """paro_plan_masked: (plan of the trainable tensors, frozen-parameter plan or None)."""
        sizes = [int(x) for x in param_sizes]
        assert len(trainable) == len(sizes)
        arr = (_i64 * max(1, len(sizes)))(*sizes)
        msk = (C.c_uint8 * max(1, len(sizes)))(*[1 if t else 0 for t in trainable])
        o = make_opts(**opts)
        ht, hf = _vp(), _vp()
        check(paro_plan_masked(ctx.h, strategy.encode(), arr, msk, len(sizes), C.byref(o), C.byref(ht), C.byref(hf)))
        out = []
        for h, sub in ((ht, [s for s, t in zip(sizes, trainable) if t]),
                       (hf, [s for s, t in zip(sizes, trainable) if not t])):
            if not h.value:
                out.append(None)
                continue
            pl = cls.__new__(cls)
            pl.ctx, pl.sizes, pl.opts, pl.h, pl.strategy = ctx, sub, o, h, strategy
            out.append(pl)
        return tuple(out)

    def __init__(self, ctx: Context, strategy: str, param_sizes, **opts):
        self.ctx = ctx
        self.sizes = [int(s) for s in param_sizes]
        arr = (_i64 * max(1, len(self.sizes)))(*self.sizes)
        self.opts = make_opts(**opts)
        h = _vp()
        check(paro_plan(ctx.h, strategy.encode(), arr, len(self.sizes), C.byref(self.opts), C.byref(h)))
        self.h = h
        self.strategy = strategy

    def info(self):
        i = paro_plan_info_t()
        check(paro_plan_info(self.h, C.byref(i)))
        return {k: getattr(i, k) for k, _ in paro_plan_info_t._fields_}

    def shard_range(self, state, rank, bucket):
        b, e = _i64(), _i64()
        check(paro_shard_range(self.h, STATE[state] if isinstance(state, str) else state, rank, bucket,
                               C.byref(b), C.byref(e)))
        return b.value, e.value

    def bucket_range(self, bucket):
        b, e = _i64(), _i64()
        check(paro_bucket_range(self.h, bucket, C.byref(b), C.byref(e)))
        return b.value, e.value

    def send_bytes(self, rank):
        a, b = _i64(), _i64()
        check(paro_rank_send_bytes(self.h, rank, C.byref(a), C.byref(b)))
        return a.value, b.value

    def accum_send_bytes(self, rank):
        """((intra, inter) per paro_accumulate call, (intra, inter) of the step after it)."""
        v = [_i64() for _ in range(4)]
        check(paro_rank_accum_send_bytes(self.h, rank, *[C.byref(x) for x in v]))
        return (v[0].value, v[1].value), (v[2].value, v[3].value)

    def gather_window(self, rank, bucket, slot=0, stream=None):
        """paro_gather_window: device address of bucket `bucket`'s full bf16 parameters."""
        out = _vp()
        check(paro_gather_window(self.h, rank, int(bucket), int(slot), stream, C.byref(out)))
        return out.value

    def gather_send_bytes(self, rank, bucket=None):
        """(intra, inter) bytes `rank` sends gathering every bucket once, or one bucket."""
        a, b = _i64(), _i64()
        if bucket is None:
            check(paro_rank_gather_send_bytes(self.h, rank, C.byref(a), C.byref(b)))
        else:
            check(paro_bucket_gather_send_bytes(self.h, rank, int(bucket), C.byref(a), C.byref(b)))
        return a.value, b.value

    def buffer(self, rank, kind):
        p = _vp()
        check(paro_buffer(self.h, rank, kind, C.byref(p)))
        return p.value

    def opt_state_init(self, rank, st, master_full_ptr=None, seed=None):
        """st: (master, m, v) device pointers, or None for a frozen-parameter plan."""
        sp = C.byref(paro_opt_state_t(*st)) if st is not None else None
        if master_full_ptr is not None:
            check(paro_opt_state_init(self.h, rank, master_full_ptr, sp))
        else:
            check(paro_opt_state_init_synth(self.h, rank, int(seed), sp))

    def synth_grads(self, rank, seed, step):
        check(paro_synth_grads(self.h, rank, int(seed), int(step)))

    def step(self, opt_states, lr, step, grads=None, params=None):
        """opt_states: list (per local rank) of (master, m, v) device pointers;
        grads / params: None (zero-copy flat buffers) or flat lists of pointers."""
        n = len(opt_states)
        sts = (paro_opt_state_t * n)(*[paro_opt_state_t(*s) for s in opt_states])
        gp = (_vp * len(grads))(*grads) if grads is not None else None
        pp = (_vp * len(params))(*params) if params is not None else None
        check(paro_step(self.h, gp, pp, sts, float(lr), int(step)))

    def step_streamed(self, opt_states, lr, step, seed=None, grad_step=None, producer=None, params=None):
        """paro_step_streamed (grad_slots plans).  producer(rank, bucket, begin, end, dst_ptr, stream_ptr)
        enqueues bucket `bucket`'s bf16 gradients into dst on that CUDA stream; None = the library's
        synthetic gradients of (seed, grad_step)."""
        n = len(opt_states)
        sts = (paro_opt_state_t * n)(*[paro_opt_state_t(*s) for s in opt_states])
        pp = (_vp * len(params))(*params) if params is not None else None
        if producer is None:
            cb = C.cast(None, PRODUCER)
        else:
            cb = PRODUCER(lambda _u, r, b, b0, b1, dst, stream: producer(r, b, b0, b1, dst, stream))
        self._producer_ref = cb      # kept alive: the library calls it from this thread during the call
        check(paro_step_streamed(self.h, cb, None, int(seed or 0), int(grad_step or 0), pp, sts, float(lr),
                                 int(step)))

    def set_param_consumer(self, consumer):
        """paro_set_param_consumer: consumer(rank, bucket, begin, end, src_ptr, stream_ptr) enqueues reads of
        bucket `bucket`'s updated bf16 parameters (the rank's P residency [begin, end)) on that CUDA stream
        during every following step; None unregisters."""
        if consumer is None:
            cb = C.cast(None, CONSUMER)
        else:
            cb = CONSUMER(lambda _u, r, b, b0, b1, src, stream: consumer(r, b, b0, b1, src, stream))
        self._consumer_ref = cb       # kept alive: the library calls it during later steps
        check(paro_set_param_consumer(self.h, cb, None))

    def accumulate(self, grads=None):
        """paro_accumulate: add one micro-batch (grads: None = the flat gradient
        buffers, else a flat list of per-parameter pointers, rank-major)."""
        gp = (_vp * len(grads))(*grads) if grads is not None else None
        check(paro_accumulate(self.h, gp))

    def stats(self):
        s = paro_step_stats_t()
        check(paro_step_stats(self.h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in paro_step_stats_t._fields_}

    def collective(self, what=0):
        check(paro_collective(self.h, int(what)))

    def profile_start(self, max_launches):
        check(paro_profile_start(self.h, int(max_launches)))

    def profile_stop(self):
        s = paro_profile_t()
        check(paro_profile_stop(self.h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in paro_profile_t._fields_}

    def close(self):
        if self.h:
            paro_plan_destroy(self.h)
            self.h = None
