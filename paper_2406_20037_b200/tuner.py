"""Thin Python binding over the C ABI (include/tuner.h): argument marshalling
only.  Every step of the hot path (sampling, dispatch, execution, verification,
timing, all-gather, Droplet Search) runs inside libdroplet_b200.so; PyTorch is
used for device memory, streams and process groups.

    t = Tuner("conv2d", shape, dtype="f32", x=x, w=w, y=y)     # measured mode
    t.sample(300); b = t.best(); rep = t.droplet(b.point, 100)   # DPAnsor
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

from . import _lib as L

PointT = Tuple[int, Tuple[int, ...]]

_GROUP_UIDS: Dict[int, object] = {}  # process group -> 128-byte NCCL unique id


@dataclass
class Sample:
    point: PointT
    cost_ns: float
    max_err: float
    status: str
    rank: int


def _point(p: PointT) -> L.Point:
    s, idx = p
    pt = L.Point()
    pt.sketch = int(s)
    pt.n = len(idx)
    if pt.n > L.MAX_KNOBS:
        raise ValueError("too many knobs")
    for i, v in enumerate(idx):
        pt.idx[i] = int(v)
    return pt


def _unpoint(pt: L.Point) -> PointT:
    return (int(pt.sketch), tuple(int(pt.idx[i]) for i in range(pt.n)))


def _sample(r: L.Result) -> Sample:
    st = L.SAMPLE_STATUS[r.status] if 0 <= r.status < len(L.SAMPLE_STATUS) else str(r.status)
    return Sample(_unpoint(r.pt), float(r.cost_ns), float(r.max_err), st, int(r.rank))


def sketches(op: str, dtype: str = "f32") -> List[int]:
    ids = (C.c_int32 * 32)()
    n = C.c_int32()
    L.check(L.lib().tuner_sketches(L.OP[op], L.DTYPE[dtype], ids, 32, C.byref(n)))
    return [ids[i] for i in range(min(n.value, 32))]


def sketch_valid(op: str, shape: Dict, sketch: int, values: Sequence[int], dtype: str = "f32") -> bool:
    """The sketch's static validity rule for a point given by knob values (no handle, no device)."""
    vals = (C.c_int32 * max(1, len(values)))(*[int(v) for v in values])
    ok = C.c_int32()
    L.check(L.lib().tuner_sketch_valid(L.OP[op], C.byref(_shape(op, shape, dtype)), sketch, vals, len(values),
                                       C.byref(ok)))
    return bool(ok.value)


def sketch_space(sketch: int) -> List[List[int]]:
    """The full compiled knob space of a sketch: one value list per knob."""
    nk = C.c_int32()
    card = (C.c_int32 * L.MAX_KNOBS)()
    vals = (C.c_int32 * (L.MAX_KNOBS * L.MAX_VALUES))()
    L.check(L.lib().tuner_sketch_space(sketch, C.byref(nk), card, vals))
    out, off = [], 0
    for d in range(nk.value):
        out.append([vals[off + i] for i in range(card[d])])
        off += card[d]
    return out


def sketch_name(sketch: int) -> str:
    s = L.lib().tuner_sketch_name(sketch)
    return s.decode() if s else None


def knob_names(sketch: int) -> List[str]:
    out, i = [], 0
    while True:
        s = L.lib().tuner_knob_name(sketch, i)
        if not s:
            return out
        out.append(s.decode())
        i += 1


def schedule(tuners: Sequence["Tuner"], weights: Sequence[float], budget: int, increment: int = 16,
             drop_frac: float = 0.01, pop: int = 64, elite: int = 16) -> List[int]:
    """Multi-layer trial budget across a model's layers (tuner_schedule); returns trials per layer."""
    n = len(tuners)
    hs = (C.c_void_p * n)(*[t._h.value for t in tuners])
    ws = (C.c_double * n)(*[float(w) for w in weights])
    out = (C.c_int64 * n)()
    L.check(L.lib().tuner_schedule(hs, n, ws, int(budget), increment, float(drop_frac), pop, elite, out))
    return [int(out[i]) for i in range(n)]


def global_launch_count() -> int:
    return int(L.lib().tuner_global_launch_count())


def rank_sum_p(a: Sequence[float], b: Sequence[float]) -> float:
    """Two-sided exact Wilcoxon rank-sum p of two timing samples (tuner_rank_sum_p)."""
    fa = (C.c_float * max(1, len(a)))(*a)
    fb = (C.c_float * max(1, len(b)))(*b)
    p = C.c_double()
    L.check(L.lib().tuner_rank_sum_p(fa, len(a), fb, len(b), C.byref(p)))
    return p.value


def probe_fp32_peak(mode: int = 1) -> Tuple[float, float]:
    """FP32 pipe peak on the current device (tuner_probe_fp32_peak): (TFLOP/s, ms).
    mode 0 = 3-register FFMA, 1 = FFMA2, 2 = immediate-operand FFMA."""
    tf, ms = C.c_double(), C.c_double()
    L.check(L.lib().tuner_probe_fp32_peak(mode, C.byref(tf), C.byref(ms)))
    return tf.value, ms.value


def _shape(op: str, shape: Dict, dtype: str) -> L.Shape:
    s = L.Shape()
    s.dtype = L.DTYPE[dtype]
    if op in ("conv2d", "depthwise_conv2d"):
        s.N, s.C, s.H, s.W = shape["N"], shape["C"], shape["H"], shape.get("W", shape["H"])
        s.K = shape["K"] if op == "conv2d" else shape.get("K", shape["C"])
        s.R, s.S = shape["R"], shape.get("S", shape["R"])
        st, pd, dl = shape.get("stride", (1, 1)), shape.get("pad", (0, 0)), shape.get("dil", (1, 1))
        s.stride_h, s.stride_w = st
        s.pad_h, s.pad_w = pd
        s.dil_h, s.dil_w = dl
    else:
        s.b = shape.get("b", 1)
        s.m, s.n, s.k = shape["m"], shape["n"], shape["k"]
    return s


def _ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


class Tuner:
    """One layer's tuner (a handle of the C library)."""

    def __init__(self, op: str, shape: Dict, *, dtype: str = "f32",
                 spaces: Optional[Sequence[Tuple[int, Sequence[Sequence[int]]]]] = None,
                 seed: int = 0, policy: str = "grow", cost_table=None,
                 x=None, w=None, y=None, y_ref=None, y_absref=None, stream=None, group=None,
                 warmup: int = 2, repeats: int = 10, number: int = 0, max_batch: int = 512,
                 verify: bool = True, timeout_ms: float = 1000.0, early_cut: float = 0.0,
                 alpha: float = 0.0, cost_samples=None, trial_log: Optional[str] = None):
        lib = L.lib()
        self._h = C.c_void_p()
        self.op = op
        if spaces is None:
            if cost_table is not None:
                raise ValueError("cost-table mode needs explicit spaces")
            spaces = [(s, sketch_space(s)) for s in sketches(op, dtype)]
        self.spaces = [(int(s), [list(map(int, v)) for v in vals]) for s, vals in spaces]
        ks = (L.KnobSpace * len(self.spaces))()
        self._keep = []
        for i, (sid, vals) in enumerate(self.spaces):
            card = (C.c_int32 * max(1, len(vals)))(*[len(v) for v in vals])
            flat = [x_ for v in vals for x_ in v]
            va = (C.c_int32 * max(1, len(flat)))(*flat)
            self._keep += [card, va]
            ks[i].sketch, ks[i].nknobs, ks[i].card, ks[i].values = sid, len(vals), card, va
        o = L.Opts()
        lib.tuner_opts_default(C.byref(o))
        o.warmup, o.repeats, o.number = warmup, repeats, number
        o.timeout_ms, o.seed, o.policy = timeout_ms, seed, L.POLICY[policy]
        o.max_batch, o.verify, o.early_cut = max_batch, int(bool(verify)), float(early_cut)
        o.alpha = float(alpha)
        if trial_log:
            self._log = str(trial_log).encode()
            o.trial_log = self._log
        if cost_table is not None:
            import numpy as np
            tab = np.ascontiguousarray(cost_table, dtype=np.float64)
            self._keep.append(tab)
            o.cost_table = tab.ctypes.data_as(C.POINTER(C.c_double))
            o.cost_table_len = tab.size
            if cost_samples is not None:
                smp = np.ascontiguousarray(cost_samples, dtype=np.float64)
                self._keep.append(smp)
                o.cost_samples = smp.ctypes.data_as(C.POINTER(C.c_double))
                o.cost_nsamp = smp.shape[1]
        else:
            if x is None or w is None or y is None:
                raise ValueError("measured mode needs device tensors x, w, y")
            o.x, o.w, o.y = _ptr(x), _ptr(w), _ptr(y)
            o.y_ref, o.y_absref = _ptr(y_ref), _ptr(y_absref)
            if stream is None:
                import torch
                stream = torch.cuda.current_stream(x.device)
            o.stream = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        self._tensors = (x, w, y, y_ref, y_absref)
        self.world, self.rank = 1, 0
        if group is not None:
            self._setup_group(o, group, cost_table is not None)
        L.check(lib.tuner_create(L.OP[op], C.byref(_shape(op, shape, dtype)), ks, len(self.spaces), C.byref(o),
                                 C.byref(self._h)))

    def _setup_group(self, o, group, table_mode):
        import torch
        import torch.distributed as dist
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        o.world, o.rank = self.world, self.rank
        backend = dist.get_backend(group)
        if self.world == 1 and backend != "nccl":
            return  # nothing to exchange (a 1-rank NCCL group still runs the collective path)
        if backend == "nccl" and not table_mode:
            # one NCCL unique id per process group: the library keeps one communicator per id,
            # shared by every tuner of the group (SPMD: every rank creates tuners in the same order)
            key = id(group)
            if key not in _GROUP_UIDS:
                uid = (C.c_char * 128)()
                if self.rank == 0:
                    L.check(L.lib().tuner_nccl_unique_id(uid))
                objs = [bytes(uid)]
                dist.broadcast_object_list(objs, src=dist.get_global_rank(group, 0), group=group)
                _GROUP_UIDS[key] = (C.c_char * 128).from_buffer_copy(objs[0])
            self._uid = _GROUP_UIDS[key]
            o.nccl_unique_id = C.cast(self._uid, C.c_void_p)
            return

        def allgather(ctx, send, recv, nbytes):  # host all-gather over the process group (e.g. gloo)
            try:
                buf = torch.frombuffer(bytearray(C.string_at(send, nbytes)), dtype=torch.uint8)
                outs = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(self.world)]
                dist.all_gather(outs, buf, group=group)
                C.memmove(recv, bytes(torch.cat(outs).numpy().tobytes()), nbytes * self.world)
                return 0
            except Exception:
                return 1
        self._cb = L.ALLGATHER_FN(allgather)
        o.allgather = self._cb

    # ------------------------------------------------------------------ API
    def sample(self, n: int) -> List[Sample]:
        out = (L.Result * max(1, n))()
        got = C.c_int32()
        L.check(L.lib().tuner_sample(self._h, n, out, C.byref(got)))
        return [_sample(out[i]) for i in range(got.value)]

    def grid(self, n: int) -> List[Sample]:
        """Grid search: the next n valid unmeasured points in enumeration order (tuner_grid)."""
        out = (L.Result * max(1, n))()
        got = C.c_int32()
        L.check(L.lib().tuner_grid(self._h, n, out, C.byref(got)))
        return [_sample(out[i]) for i in range(got.value)]

    def evolve(self, n: int, pop: int = 64, elite: int = 16) -> List[Sample]:
        """Ansor-style evolutionary exploration (tuner_evolve)."""
        out = (L.Result * max(1, n))()
        got = C.c_int32()
        L.check(L.lib().tuner_evolve(self._h, n, pop, elite, out, C.byref(got)))
        return [_sample(out[i]) for i in range(got.value)]

    def measure(self, points: Sequence[PointT]) -> List[Sample]:
        n = len(points)
        pts = (L.Point * max(1, n))(*[_point(p) for p in points])
        out = (L.Result * max(1, n))()
        L.check(L.lib().tuner_measure(self._h, pts, n, out))
        return [_sample(out[i]) for i in range(n)]

    def droplet(self, start: PointT, budget: int = 100) -> Dict:
        rep = L.DropletReport()
        cap = 4096
        traj = (L.Point * cap)()
        L.check(L.lib().tuner_droplet(self._h, C.byref(_point(start)), budget, traj, cap, C.byref(rep)))
        return {"best": _unpoint(rep.best), "best_cost": float(rep.best_cost), "trials_used": rep.trials_used,
                "rounds": rep.rounds, "converged": bool(rep.converged),
                "traj": [_unpoint(traj[i]) for i in range(min(rep.traj_len, cap))]}

    def timings(self, p: PointT) -> List[float]:
        """The repeat timings (ns per launch) behind a measured point's cost."""
        buf = (C.c_float * 16)()
        n = C.c_int32()
        L.check(L.lib().tuner_timings(self._h, C.byref(_point(p)), buf, 16, C.byref(n)))
        return [float(buf[i]) for i in range(n.value)]

    def best(self) -> Sample:
        r = L.Result()
        L.check(L.lib().tuner_best(self._h, C.byref(r)))
        return _sample(r)

    def best_of_sketch(self, sketch: int) -> Optional[Sample]:
        """First argmin among one sketch's measured points (tuner_best_of_sketch); None if it has
        no finite measurement."""
        r = L.Result()
        st = L.lib().tuner_best_of_sketch(self._h, sketch, C.byref(r))
        if st == L.ESTATE:
            return None
        L.check(st)
        return _sample(r)

    def history(self) -> List[Sample]:
        n = C.c_int64()
        L.check(L.lib().tuner_history(self._h, None, 0, C.byref(n)))
        out = (L.Result * max(1, n.value))()
        L.check(L.lib().tuner_history(self._h, out, n.value, C.byref(n)))
        return [_sample(out[i]) for i in range(n.value)]

    def valid(self, p: PointT) -> bool:
        v = C.c_int32()
        L.check(L.lib().tuner_point_valid(self._h, C.byref(_point(p)), C.byref(v)))
        return bool(v.value)

    def run(self, cfg: PointT, x, w, y, stream=None):
        b = L.Buffers(_ptr(x), _ptr(w), _ptr(y))
        s = 0 if stream is None else (stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
        L.check(L.lib().kernel_run(self._h, C.byref(_point(cfg)), C.byref(b), C.c_void_p(s)))

    def reference(self, x, w, y_ref, y_absref, stream=None):
        b = L.Buffers(_ptr(x), _ptr(w), 0)
        s = 0 if stream is None else (stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
        L.check(L.lib().tuner_reference(self._h, C.byref(b), C.c_void_p(_ptr(y_ref)), C.c_void_p(_ptr(y_absref)),
                                        C.c_void_p(s)))

    def stats(self) -> Dict:
        s = L.Stats()
        L.check(L.lib().tuner_get_stats(self._h, C.byref(s)))
        return {"kernel_launches": s.kernel_launches, "candidates": s.candidates, "collectives": s.collectives,
                "batches": s.batches, "measure_wall_ns": s.measure_wall_ns, "early_cut": s.early_cut,
                "light": s.light, "precise": s.precise, "calibrations": s.calibrations, "replayed": s.replayed}

    def values(self, p: PointT) -> List[int]:
        sid, idx = p
        vals = dict(self.spaces)[sid]
        return [vals[d][i] for d, i in enumerate(idx)]

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            L.lib().tuner_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
