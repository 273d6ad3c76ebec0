"""Thin Python binding over the C ABI (same names, argument marshalling only).

Every step of the BOCD hot path runs in the CUDA kernels of libfalcon_bocd.so;
PyTorch supplies device memory and streams.  Nothing here computes.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native as N

EVENT_DTYPE = np.dtype([("series", np.int64), ("t", np.int64), ("cp_index", np.int64),
                        ("flags", np.uint32), ("reserved", np.uint32), ("p_new", np.float64)])


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _ld(x):
    """Row stride of a 2-D row-major array (a single row may carry any stride)."""
    return x.stride(0) if x.shape[0] > 1 else max(x.stride(0), x.shape[1])


def _stream_ptr(stream, device=None):
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return ctypes.c_void_p(stream.cuda_stream)


class DrainTicket:
    """An enqueued asynchronous drain (BocdBatch.changepoints_async)."""

    def __init__(self, batch, buf, meta, event, stream, device_out=False):
        self._batch, self._buf, self._meta, self._event, self._stream = batch, buf, meta, event, stream
        self._device_out = device_out

    def result(self):
        """Waits for the drain; returns (events, dropped) as BocdBatch.changepoints()."""
        self._event.synchronize()
        total, ovf, err, drained = (int(v) for v in self._meta.tolist())
        self._batch._ev_hint = max(self._batch._ev_hint, total)
        if not drained:  # capacity too small or a sticky error: nothing changed, drain (or raise) now
            return self._batch.changepoints(self._stream, device_out=self._device_out)
        if self._device_out:
            return self._buf[:total].clone(), bool(ovf)
        return self._buf[:total].numpy().reshape(-1).view(EVENT_DTYPE).copy(), bool(ovf)


class BocdBatch:
    """falcon_bocd_create / _update_chunk / _changepoints / _read_posterior / _destroy."""

    N_TICKETS = 4  # asynchronous drains that may be outstanding at once

    def __init__(self, n_series: int, R: int = 1024, hazard: float = 1.0 / 250.0,
                 kappa0: float = 1.0, alpha0: float = 1.0, mu0=0.0, beta0=1.0,
                 prior_first_obs: bool = False, prior_cov: float = 0.05, threshold: float = 0.9,
                 trunc_mode: str | int = "merge", event_mask: int = N.EV_PROB,
                 event_capacity: int = 64, device: int | None = None, series_base: int = 0):
        L = N.lib()
        cfg = N.Config()
        N.check(L.falcon_bocd_config_init(ctypes.byref(cfg)))
        if device is None:
            device = torch.cuda.current_device()
        cfg.n_series = int(n_series)
        cfg.R = int(R)
        cfg.hazard = float(hazard)
        cfg.kappa0 = float(kappa0)
        cfg.alpha0 = float(alpha0)
        keep = []
        for name in ("mu0", "beta0"):
            val = mu0 if name == "mu0" else beta0
            arr = np.asarray(val, dtype=np.float64)
            if arr.ndim == 0:
                setattr(cfg, name, None)
                setattr(cfg, name + "_scalar", float(arr))
            else:
                arr = np.ascontiguousarray(arr.reshape(int(n_series)))
                keep.append(arr)
                setattr(cfg, name, arr.ctypes.data)
        cfg.prior_first_obs = int(bool(prior_first_obs))
        cfg.prior_cov = float(prior_cov)
        cfg.threshold = float(threshold)
        if isinstance(trunc_mode, str):
            trunc_mode = {"merge": N.TRUNC_MERGE, "drop": N.TRUNC_DROP}[trunc_mode.lower()]
        cfg.trunc_mode = int(trunc_mode)
        cfg.event_mask = int(event_mask)
        cfg.event_capacity = int(event_capacity)
        cfg.device = int(device)
        cfg.series_base = int(series_base)
        h = ctypes.c_void_p()
        N.check(L.falcon_bocd_create(ctypes.byref(cfg), ctypes.byref(h)), None)
        self._h = h
        self.n_series, self.R, self.device = int(n_series), int(R), torch.device("cuda", int(device))
        self.event_capacity = int(event_capacity)
        self._evbufs = {}
        self._ev_hint = min(self.n_series * self.event_capacity, 4096)
        self._metas = [torch.zeros(4, dtype=torch.int64, pin_memory=True) for _ in range(self.N_TICKETS)]
        self._ticket_slot = 0

    # -- hot path ---------------------------------------------------------------
    def update_chunk(self, x: torch.Tensor, outputs: bool = False, stream=None):
        """Absorb x[:, :T] (device fp64, row stride x.stride(0)).  With outputs=True returns
        (map_rl int32, p_new fp64, log_z fp64), each [S][T] on the device."""
        assert x.is_cuda and x.dtype == torch.float64 and x.dim() == 2 and x.stride(1) == 1
        assert x.shape[0] == self.n_series
        T = x.shape[1]
        outs, res = None, None
        if outputs:
            res = (torch.empty((self.n_series, T), dtype=torch.int32, device=x.device),
                   torch.empty((self.n_series, T), dtype=torch.float64, device=x.device),
                   torch.empty((self.n_series, T), dtype=torch.float64, device=x.device))
            outs = N.StepOut(res[0].data_ptr(), res[1].data_ptr(), res[2].data_ptr(), T)
        N.check(N.lib().falcon_bocd_update_chunk(self._h, _ptr(x), _ld(x), T,
                                                 ctypes.byref(outs) if outs else None,
                                                 _stream_ptr(stream, self.device)), self._h)
        return res

    def update_chunk_host(self, x: np.ndarray | torch.Tensor, outputs: bool = False, stream=None):
        """Absorb HOST x[S][T] (pinned recommended); copies happen inside the library."""
        if isinstance(x, torch.Tensor):
            assert x.device.type == "cpu" and x.dtype == torch.float64 and x.stride(1) == 1
            ptr, ld, T = x.data_ptr(), _ld(x), x.shape[1]
        else:
            assert x.dtype == np.float64 and x.strides[1] == 8
            ptr, ld, T = x.ctypes.data, (x.strides[0] // 8 if x.shape[0] > 1 else x.shape[1]), x.shape[1]
        outs, res = None, None
        if outputs:
            res = (np.empty((self.n_series, T), np.int32), np.empty((self.n_series, T)),
                   np.empty((self.n_series, T)))
            outs = N.StepOut(res[0].ctypes.data, res[1].ctypes.data, res[2].ctypes.data, T)
        N.check(N.lib().falcon_bocd_update_chunk_host(self._h, ctypes.c_void_p(ptr), ld, T,
                                                      ctypes.byref(outs) if outs else None,
                                                      _stream_ptr(stream, self.device)), self._h)
        return res

    def _event_buffer(self, where: str, need: int, slot: int = 0):
        """Cached drain buffer (uint8 [cap, 40]): 'host' = page-locked (the gather kernel writes it
        directly), 'device' = this handle's device.  Grows geometrically."""
        key = (where, slot)
        buf = self._evbufs.get(key)
        if buf is None or buf.shape[0] < need:
            cap = max(need, 2 * (buf.shape[0] if buf is not None else 0), 1024)
            if where == "host":
                buf = torch.empty((cap, EVENT_DTYPE.itemsize), dtype=torch.uint8, pin_memory=True)
            else:
                buf = torch.empty((cap, EVENT_DTYPE.itemsize), dtype=torch.uint8, device=self.device)
            self._evbufs[key] = buf
        return buf

    def drain_into(self, out: torch.Tensor, meta: torch.Tensor, stream=None):
        """Enqueue a drain into caller-owned buffers (falcon_bocd_changepoints_async): out uint8
        [capacity, 40] and meta int64 [4], each device memory or page-locked host memory.  No
        synchronisation; after the stream reaches it, meta = (total, overflow, error bits,
        drained) and out[:total] holds the events when drained == 1."""
        assert out.dtype == torch.uint8 and out.dim() == 2 and out.shape[1] == EVENT_DTYPE.itemsize
        assert meta.dtype == torch.int64 and meta.numel() >= 4 and meta.is_contiguous()
        N.check(N.lib().falcon_bocd_changepoints_async(self._h, ctypes.c_void_p(out.data_ptr()), out.shape[0],
                                                       ctypes.c_void_p(meta.data_ptr()),
                                                       _stream_ptr(stream, self.device)), self._h)

    def reserve_events(self, n: int, device_out: bool = False):
        """Pre-allocate every drain buffer for n events (keeps allocations out of a timed loop)."""
        where = "device" if device_out else "host"
        for slot in [-1, *range(self.N_TICKETS)]:
            self._event_buffer(where, n, slot)
        self._ev_hint = max(self._ev_hint, n // 2)

    def changepoints(self, stream=None, device_out: bool = False):
        """Drain buffered events in (series, t) order (falcon_bocd_changepoints).  Returns
        (events, dropped) where events is a numpy structured array (host) or a uint8 device
        tensor of 40-B records."""
        L = N.lib()
        n = ctypes.c_int64()
        need = self._ev_hint
        while True:
            buf = self._event_buffer("device" if device_out else "host", need, slot=-1)
            rc = L.falcon_bocd_changepoints(self._h, ctypes.c_void_p(buf.data_ptr()), buf.shape[0],
                                            ctypes.byref(n), _stream_ptr(stream, self.device))
            if rc == N.FALCON_EINVAL and n.value > buf.shape[0]:
                need = int(n.value)  # nothing was drained: retry with room for every event
                continue
            N.check(rc, self._h)
            break
        k = int(n.value)
        self._ev_hint = max(self._ev_hint, k)
        if device_out:
            return buf[:k].clone(), rc == N.FALCON_WARN_EVENTS_DROPPED
        return buf[:k].numpy().reshape(-1).view(EVENT_DTYPE).copy(), rc == N.FALCON_WARN_EVENTS_DROPPED

    def changepoints_async(self, stream=None, device_out: bool = False):
        """Enqueue a drain on `stream` without synchronising (falcon_bocd_changepoints_async);
        the events land in page-locked host memory (or, device_out, in device memory).  Returns
        a DrainTicket whose result() waits for it and returns (events, dropped) like
        changepoints().  Up to N_TICKETS tickets may be outstanding at a time."""
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        slot = self._ticket_slot
        self._ticket_slot = (slot + 1) % self.N_TICKETS
        buf = self._event_buffer("device" if device_out else "host", 2 * self._ev_hint, slot)
        meta = self._metas[slot]
        N.check(N.lib().falcon_bocd_changepoints_async(self._h, ctypes.c_void_p(buf.data_ptr()), buf.shape[0],
                                                       ctypes.c_void_p(meta.data_ptr()),
                                                       ctypes.c_void_p(st.cuda_stream)), self._h)
        ev = torch.cuda.Event()
        ev.record(st)
        return DrainTicket(self, buf, meta, ev, stream, device_out)

    def read_posterior(self, s0: int = 0, count: int | None = None, stream=None):
        """(logR, mu, beta) as device tensors [count][R] in run-length order."""
        count = self.n_series - s0 if count is None else count
        out = [torch.empty((count, self.R), dtype=torch.float64, device=self.device) for _ in range(3)]
        N.check(N.lib().falcon_bocd_read_posterior(self._h, s0, count, _ptr(out[0]), _ptr(out[1]),
                                                   _ptr(out[2]), _stream_ptr(stream, self.device)), self._h)
        return tuple(out)

    def set_schedule(self, schedule: str):
        """Kernel schedule of later calls: 'auto', 'persistent' (every call of <= 64 steps),
        'one_unit' or 'one_unit_packed' (never the balanced one-CTA-per-SM wave)
        (falcon_bocd_set_schedule; a test hook: results are bit-identical)."""
        code = {"auto": 0, "persistent": 1, "one_unit": 2, "one_unit_packed": 3}[schedule]
        N.check(N.lib().falcon_bocd_set_schedule(self._h, code), self._h)

    @property
    def steps(self) -> int:
        t = ctypes.c_int64()
        N.check(N.lib().falcon_bocd_steps(self._h, ctypes.byref(t)), self._h)
        return int(t.value)

    def kernel_shape(self):
        a, b, c = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        N.check(N.lib().falcon_bocd_kernel_shape(self._h, ctypes.byref(a), ctypes.byref(b),
                                                 ctypes.byref(c)), self._h)
        return int(a.value), int(b.value), int(c.value)

    def close(self):
        if getattr(self, "_h", None):
            rc = N.lib().falcon_bocd_destroy(self._h)
            self._h = None
            if rc not in (N.FALCON_OK, N.FALCON_ENONFINITE):  # ENONFINITE was reported earlier
                N.check(rc, None)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                N.lib().falcon_bocd_destroy(self._h)
                self._h = None
        except Exception:
            pass


VERIFIED_DTYPE = np.dtype([("series", np.int64), ("t", np.int64), ("cp_index", np.int64), ("status", np.int32),
                           ("n_before", np.int32), ("n_after", np.int32), ("reserved", np.int32),
                           ("mean_before", np.float64), ("mean_after", np.float64)])
FAILSLOW_DTYPE = np.dtype([("series", np.int64), ("onset", np.int64), ("recovery", np.int64),
                           ("severity", np.float64)])


def verify_changepoints(x, events, t_lo: int = 0, series_base: int = 0, window: int = 20,
                        rel_threshold: float = 0.10, stream=None):
    """Change-point verification (N1, falcon_verify_changepoints): x is a CUDA fp64 tensor
    [n_series][T] (row k = global series series_base + k, column j = global step t_lo + j);
    events a host EVENT_DTYPE array (e.g. from BocdBatch.changepoints()).  Returns a host
    VERIFIED_DTYPE array, one record per event."""
    assert x.is_cuda and x.dtype == torch.float64 and x.dim() == 2 and x.stride(1) == 1
    ev = np.ascontiguousarray(events, dtype=EVENT_DTYPE)
    n = len(ev)
    if n == 0:
        return np.empty(0, dtype=VERIFIED_DTYPE)
    st = stream if stream is not None else torch.cuda.current_stream(x.device)
    with torch.cuda.stream(st):  # upload, kernel and read-back all ordered on `st`
        ev_d = torch.from_numpy(ev.view(np.uint8).reshape(n, EVENT_DTYPE.itemsize)).to(x.device)
        out_d = torch.empty((n, VERIFIED_DTYPE.itemsize), dtype=torch.uint8, device=x.device)
        N.check(N.lib().falcon_verify_changepoints(_ptr(x), _ld(x), x.shape[0], series_base, t_lo,
                                                   x.shape[1], _ptr(ev_d), n, window, rel_threshold,
                                                   _ptr(out_d), ctypes.c_void_p(st.cuda_stream)))
        return out_d.cpu().numpy().reshape(-1).view(VERIFIED_DTYPE).copy()


def pair_failslow(verified, device=None, stream=None):
    """Fail-slow pairing (N1, falcon_pair_failslow) of a VERIFIED_DTYPE array in (series, t)
    order.  Returns a host FAILSLOW_DTYPE array in (series, onset) order."""
    v = np.ascontiguousarray(verified, dtype=VERIFIED_DTYPE)
    n = len(v)
    if n == 0:
        return np.empty(0, dtype=FAILSLOW_DTYPE)
    dev = device or torch.device("cuda", torch.cuda.current_device())
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    with torch.cuda.stream(st):
        v_d = torch.from_numpy(v.view(np.uint8).reshape(n, VERIFIED_DTYPE.itemsize)).to(dev)
        cap = int((v["status"] == N.CP_DEGRADE).sum())
        out_d = torch.empty((max(cap, 1), FAILSLOW_DTYPE.itemsize), dtype=torch.uint8, device=dev)
        n_out = ctypes.c_int64()
        N.check(N.lib().falcon_pair_failslow(_ptr(v_d), n, _ptr(out_d), cap, ctypes.byref(n_out),
                                             ctypes.c_void_p(st.cuda_stream)))
        return out_d[: n_out.value].cpu().numpy().reshape(-1).view(FAILSLOW_DTYPE).copy()


def classify_groups(times, factor: float = 1.1, stream=None):
    """Suspicious-group classification (N4, falcon_classify_groups): times is a CUDA fp64
    tensor [n_batches][n_groups] of per-group transfer times.  Returns (suspicious: bool
    tensor [n_batches][n_groups], median: fp64 tensor [n_batches]) on the device."""
    assert times.is_cuda and times.dtype == torch.float64 and times.dim() == 2 and times.stride(1) == 1
    B, G_ = times.shape
    flags = torch.empty((B, G_), dtype=torch.uint8, device=times.device)
    med = torch.empty(B, dtype=torch.float64, device=times.device)
    N.check(N.lib().falcon_classify_groups(_ptr(times), B, G_, _ld(times), factor, _ptr(flags), _ptr(med),
                                           _stream_ptr(stream)))
    return flags.bool(), med


def detect_period(codes, k_max: int, M: float = 0.95, with_acf: bool = False, stream=None):
    """ACF period detection (N2, falcon_detect_period): codes is a CUDA int32 tensor [S][L].
    Returns period (int32 [S]: 0 = none, -1 = zero-variance window) and, with_acf, the ACF
    [S][k_max] (device tensors).  Needs L >= 2 k_max (FalconError EINVAL otherwise)."""
    assert codes.is_cuda and codes.dtype == torch.int32 and codes.dim() == 2 and codes.stride(1) == 1
    S, L = codes.shape
    period = torch.empty(S, dtype=torch.int32, device=codes.device)
    acf = torch.empty((S, k_max), dtype=torch.float64, device=codes.device) if with_acf else None
    N.check(N.lib().falcon_detect_period(_ptr(codes), S, L, _ld(codes), k_max, M, _ptr(acf), _ptr(period),
                                         _stream_ptr(stream)))
    return (period, acf) if with_acf else period


def iteration_times(ts, period, stream=None):
    """Iteration times from call timestamps (N2, falcon_iteration_times): ts CUDA fp64 [S][n],
    period int32 [S].  Returns (times fp64 [S][n-1], counts int32 [S]); row s is valid up to
    counts[s]."""
    assert ts.is_cuda and ts.dtype == torch.float64 and ts.dim() == 2 and ts.stride(1) == 1
    S, n = ts.shape
    st = stream if stream is not None else torch.cuda.current_stream(ts.device)
    with torch.cuda.stream(st):  # temporaries allocated on `st`: reused only after the kernel in stream order
        per = period.to(device=ts.device, dtype=torch.int32).contiguous()
        out = torch.zeros((S, max(n - 1, 1)), dtype=torch.float64, device=ts.device)
        cnt = torch.empty(S, dtype=torch.int32, device=ts.device)
        N.check(N.lib().falcon_iteration_times(_ptr(ts), S, n, _ld(ts), _ptr(per), _ptr(out), out.stride(0),
                                               _ptr(cnt), ctypes.c_void_p(st.cuda_stream)))
    return out, cnt


def predictive_constants(R: int, kappa0: float, alpha0: float):
    """Host-only table (c_r, alpha_r, g_r, 1/(kappa_r+1)) used by the kernels."""
    out = [np.empty(R) for _ in range(4)]
    N.check(N.lib().falcon_bocd_predictive_constants(int(R), float(kappa0), float(alpha0),
                                                     *[o.ctypes.data for o in out]))
    return tuple(out)


class DeviceTrace:
    """Device copy of a tracegen.TraceSpec, for falcon_trace_generate."""

    def __init__(self, spec, device):
        dev = torch.device(device)
        self.spec = spec
        t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt).to(dev)
        self._b = t(spec.b, torch.float64)
        self._sigma = t(spec.sigma, torch.float64)
        self._off = t(spec.ep_off, torch.int64)
        E = max(1, len(spec.ep_start))
        pad = lambda a, dt: t(np.resize(a, E) if len(a) else np.zeros(E), dt)
        self._st = pad(spec.ep_start, torch.int64)
        self._en = pad(spec.ep_end, torch.int64)
        self._ls = pad(spec.ep_logsev, torch.float64)
        self.c = N.TraceSpecC(spec.seed, spec.n_series, spec.gamma, self._b.data_ptr(),
                              self._sigma.data_ptr(), self._off.data_ptr(), self._st.data_ptr(),
                              self._en.data_ptr(), self._ls.data_ptr())

    def generate(self, out: torch.Tensor, s0: int, t0: int, stream=None):
        """out[i, j] = x(s0 + i, t0 + j) (device fp64 [count][T] with row stride out.stride(0))."""
        assert out.is_cuda and out.dtype == torch.float64 and out.stride(1) == 1
        N.check(N.lib().falcon_trace_generate(ctypes.byref(self.c), _ptr(out), out.stride(0), s0,
                                              out.shape[0], t0, out.shape[1], _stream_ptr(stream)))
        return out
