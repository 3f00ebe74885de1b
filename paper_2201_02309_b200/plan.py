"""Python face of the C ABI: `Plan` wraps katsevich_plan_* with the same names.

PyTorch is used only for device memory (workspace, outputs) and stream
handles; all arithmetic runs in libkatsevich.so's sm_100a kernels.
"""
from __future__ import annotations

import contextlib
import ctypes
import warnings

import numpy as np

from ._lib import (KATS_ERR_NO_DEVICE, KATS_OK, KATS_WARN_TD_NOT_COVERED, KatsevichError,
                   KatsevichGeometry, KatsevichStats, lib)

STAGES = ("K12_deriv_fwd_rebin", "K3_hilbert", "K4_bwd_rebin_cos", "K5_backproject", "fixup", "other")


def geometry_from_config(cfg: dict) -> KatsevichGeometry:
    """Build the C geometry from a config dict (synth/configs.py keys)."""
    return KatsevichGeometry(
        R=cfg["R"], D=cfg["D"], pitch=cfg["P"], lambda0=cfg.get("lambda0", 0.0), z0=cfg.get("z0", 0.0),
        r_fov=cfg.get("r_fov", 0.0), n_rows=cfg["n_rows"], d_w=cfg["d_w"], n_cols=cfg["n_cols"],
        d_alpha=cfg["d_alpha"], alpha_offset=cfg.get("alpha_offset", 0.0),
        views_per_turn=cfg["views_per_turn"], nx=cfg["nx"], ny=cfg["ny"], dx=cfg["dx"],
        dy=cfg.get("dy", cfg["dx"]), nz_per_pitch=cfg["nz"], n_psi=cfg.get("n_psi", 0), flags=cfg.get("flags", 0))


def _stream_handle(stream):
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


class Plan:
    """katsevich_plan: geometry + periodic tables (host double, device fp32)."""

    def __init__(self, geometry, device: int = 0):
        if isinstance(geometry, dict):
            geometry = geometry_from_config(geometry)
        self.geometry = geometry
        self.device = device
        self._h = ctypes.c_void_p()
        rc = lib().katsevich_plan_create(ctypes.byref(geometry), device, ctypes.byref(self._h))
        if rc != KATS_OK:
            raise KatsevichError(rc, "katsevich_plan_create")
        self.td_covered = None
        self._ws = None
        self._ws_home = self._ws_last = None
        self._dev = None
        self._ws_graph = []                    # workspaces a captured CUDA graph uses

    # -- lifecycle ---------------------------------------------------------
    def _check(self, rc, what=""):
        if rc < 0:
            raise KatsevichError(rc, lib().katsevich_last_error_detail(self._h).decode() or what)
        return rc

    def precompute(self, stream=None):
        s = ctypes.c_void_p(0) if self.device < 0 else _stream_handle(stream)
        rc = self._check(lib().katsevich_precompute(self._h, s))
        self.td_covered = rc != KATS_WARN_TD_NOT_COVERED
        if not self.td_covered:
            warnings.warn("detector rows do not cover the Tam-Danielsson window")
        return rc

    def close(self):
        if self._h:
            lib().katsevich_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- queries -----------------------------------------------------------
    def pitch_views(self, pitch: int = 0):
        fv, nv = ctypes.c_int64(), ctypes.c_int32()
        self._check(lib().katsevich_pitch_views(self._h, pitch, ctypes.byref(fv), ctypes.byref(nv)))
        return fv.value, nv.value

    def scan_views(self, first_pitch: int, n_pitches: int):
        fv, nv = ctypes.c_int64(), ctypes.c_int64()
        self._check(lib().katsevich_scan_views(self._h, first_pitch, n_pitches, ctypes.byref(fv), ctypes.byref(nv)))
        return fv.value, nv.value

    def workspace_bytes(self, n_pitches: int = 1, host: bool = False) -> int:
        b = ctypes.c_size_t()
        f = lib().katsevich_workspace_bytes_host if host else lib().katsevich_workspace_bytes
        self._check(f(self._h, n_pitches, ctypes.byref(b)))
        return b.value

    def table_info(self):
        n, lo, hi = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64()
        self._check(lib().katsevich_table_info(self._h, ctypes.byref(n), ctypes.byref(lo), ctypes.byref(hi)))
        return dict(n_psi=n.value, bp_lo=lo.value, bp_hi=hi.value)

    def filtered_grid(self):
        """(rows, cols) of the filtered data and the tables: the detector, or for the half-sample
        derivative (KATS_FLAG_HALF_SAMPLE) the half-shifted grid with one row and column fewer."""
        g = self.geometry
        h = 1 if g.flags & 1 else 0
        return g.n_rows - h, g.n_cols - h

    def export_tables(self):
        g = self.geometry
        nr_f, nc_f = self.filtered_grid()
        info = self.table_info()
        nvox = (g.nz_per_pitch, g.ny, g.nx)
        out = dict(pi_first=np.empty(nvox, np.int32), pi_last=np.empty(nvox, np.int32),
                   w_first=np.empty(nvox), w_last=np.empty(nvox),
                   fr_idx=np.empty((info["n_psi"], nc_f), np.int32), fr_frac=np.empty((info["n_psi"], nc_f)),
                   br_idx=np.empty((nr_f, nc_f), np.int32), br_frac=np.empty((nr_f, nc_f)))
        P32, PD = ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_double)
        self._check(lib().katsevich_export_tables(
            self._h, out["pi_first"].ctypes.data_as(P32), out["pi_last"].ctypes.data_as(P32),
            out["w_first"].ctypes.data_as(PD), out["w_last"].ctypes.data_as(PD),
            out["fr_idx"].ctypes.data_as(P32), out["fr_frac"].ctypes.data_as(PD),
            out["br_idx"].ctypes.data_as(P32), out["br_frac"].ctypes.data_as(PD)))
        return out

    # -- device entry points (torch tensors for memory) --------------------
    @contextlib.contextmanager
    def _ws_use(self, nbytes: int, stream):
        """The plan's one cached workspace for a call on `stream`.  Calls may come on different
        streams (the default stream, a capture stream): a call on another stream than the
        workspace's previous use first waits for that stream (an event recorded there at the switch,
        so same-stream calls pay nothing), and the workspace is marked in use on every stream it ran
        on, so the caching allocator does not hand it out while a kernel still reads it.  Not while
        a CUDA graph is being captured (torch.cuda.graph synchronises the device on entry): a
        captured graph keeps using this workspace, so it is then held for the plan's lifetime (a
        later, larger workspace does not free it), and eager calls on the plan must not run
        concurrently with the graph's replays."""
        import torch
        if self._dev is None:
            self._dev = torch.device("cuda", self.device)
        dev = self._dev
        if stream is None:
            st = torch.cuda.current_stream(dev)
        elif isinstance(stream, int):
            st = torch.cuda.ExternalStream(stream, device=dev)
        else:
            st = stream
        capturing = torch.cuda.is_current_stream_capturing()
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
            self._ws_home = torch.cuda.current_stream(dev)
            self._ws_last = None
        if not capturing:
            if self._ws_last is not None and self._ws_last != st:
                ev = torch.cuda.Event()
                ev.record(self._ws_last)
                st.wait_event(ev)
            if st != self._ws_home:
                self._ws.record_stream(st)
        if capturing and not any(w is self._ws for w in self._ws_graph):
            self._ws_graph.append(self._ws)
        yield self._ws
        if not capturing:
            self._ws_last = st

    def _vol_shape(self, n):
        g = self.geometry
        return (n * g.nz_per_pitch, g.ny, g.nx)

    def reconstruct(self, sino, sino_first_view: int, first_pitch: int = 0, n_pitches: int = 1,
                    out=None, stream=None):
        """sino: cuda float32 tensor [views][rows][cols] holding views from sino_first_view."""
        import torch
        assert sino.is_cuda and sino.dtype == torch.float32 and sino.is_contiguous()
        if out is None:
            out = torch.empty(self._vol_shape(n_pitches), dtype=torch.float32, device=sino.device)
        nb = self.workspace_bytes(n_pitches)
        with self._ws_use(nb, stream) as ws:
            self._check(lib().katsevich_reconstruct(self._h, _ptr(sino), sino_first_view, sino.shape[0],
                                                    first_pitch, n_pitches, _ptr(out), _ptr(ws), ws.numel(),
                                                    _stream_handle(stream)))
        return out

    def reconstruct_grouped(self, sino, sino_first_view: int, first_pitch: int, n_pitches: int, groups: int,
                            group_events=None, out=None, stream=None):
        """katsevich_reconstruct_grouped: one filter pass, then the backprojection in `groups`
        launches over consecutive pitch groups; group_events[i] (torch.cuda.Event, already
        created) is recorded on `stream` when group i's slices are written."""
        import torch
        assert sino.is_cuda and sino.dtype == torch.float32 and sino.is_contiguous()
        if out is None:
            out = torch.empty(self._vol_shape(n_pitches), dtype=torch.float32, device=sino.device)
        evs = None
        if group_events is not None:
            assert len(group_events) == groups
            assert all(e is None or e.cuda_event for e in group_events), "record each event once to create it"
            evs = (ctypes.c_void_p * groups)(*[ctypes.c_void_p(e.cuda_event) if e is not None else None
                                               for e in group_events])
        with self._ws_use(self.workspace_bytes(n_pitches), stream) as ws:
            self._check(lib().katsevich_reconstruct_grouped(self._h, _ptr(sino), sino_first_view, sino.shape[0],
                                                            first_pitch, n_pitches, _ptr(out), _ptr(ws), ws.numel(),
                                                            _stream_handle(stream), groups, evs))
        return out

    def reconstruct_batch(self, slabs, out=None, stream=None):
        """slabs: cuda float32 [B][n_views][rows][cols] of pitch-0 slabs."""
        import torch
        B = slabs.shape[0]
        assert slabs.is_cuda and slabs.dtype == torch.float32 and slabs.is_contiguous()
        assert slabs.shape[1] == self.pitch_views(0)[1]
        if out is None:
            g = self.geometry
            out = torch.empty((B, g.nz_per_pitch, g.ny, g.nx), dtype=torch.float32, device=slabs.device)
        with self._ws_use(self.workspace_bytes(B), stream) as ws:
            self._check(lib().katsevich_reconstruct_batch(self._h, _ptr(slabs), B, _ptr(out), _ptr(ws), ws.numel(),
                                                          _stream_handle(stream)))
        return out

    def reconstruct_batch_host(self, slabs_host, out_host=None, stream=None):
        """Host (numpy or pinned torch CPU) slabs [B][n_views][rows][cols] in, host volumes
        [B][nz][ny][nx] out; copies overlapped with the kernels inside the call."""
        import torch
        if isinstance(slabs_host, np.ndarray):
            slabs_host = torch.from_numpy(np.ascontiguousarray(slabs_host, dtype=np.float32))
        B = slabs_host.shape[0]
        assert slabs_host.shape[1] == self.pitch_views(0)[1]
        g = self.geometry
        if out_host is None:
            out_host = torch.empty((B, g.nz_per_pitch, g.ny, g.nx), dtype=torch.float32)
        b = ctypes.c_size_t()
        self._check(lib().katsevich_workspace_bytes_batch_host(self._h, B, ctypes.byref(b)))
        with self._ws_use(b.value, stream) as ws:
            self._check(lib().katsevich_reconstruct_batch_host(self._h, _ptr(slabs_host), B, _ptr(out_host), _ptr(ws),
                                                               ws.numel(), _stream_handle(stream)))
        return out_host

    def reconstruct_host(self, sino_host, sino_first_view: int, first_pitch: int = 0, n_pitches: int = 1,
                         out_host=None, stream=None):
        """Host (numpy or pinned torch CPU) sinogram in, host volume out; copies inside the call."""
        import torch
        if isinstance(sino_host, np.ndarray):
            sino_host = torch.from_numpy(np.ascontiguousarray(sino_host, dtype=np.float32))
        if out_host is None:
            out_host = torch.empty(self._vol_shape(n_pitches), dtype=torch.float32)
        with self._ws_use(self.workspace_bytes(n_pitches, host=True), stream) as ws:
            self._check(lib().katsevich_reconstruct_host(self._h, _ptr(sino_host), sino_first_view, sino_host.shape[0],
                                                         first_pitch, n_pitches, _ptr(out_host), _ptr(ws), ws.numel(),
                                                         _stream_handle(stream)))
        return out_host

    def adjoint_workspace_bytes(self, n_pitches: int = 1) -> int:
        b = ctypes.c_size_t()
        self._check(lib().katsevich_adjoint_workspace_bytes(self._h, n_pitches, ctypes.byref(b)))
        return b.value

    def adjoint(self, vol, sino_first_view: int, n_views: int, first_pitch: int = 0, n_pitches: int = 1,
                out=None, stream=None):
        """Transpose of reconstruct() (katsevich_adjoint): vol, a cuda float32 tensor
        [n_pitches*nz][ny][nx] -> sinogram adjoint [n_views][rows][cols] for views
        from sino_first_view (0 outside the pitches' slabs)."""
        import torch
        assert vol.is_cuda and vol.dtype == torch.float32 and vol.is_contiguous()
        g = self.geometry
        if out is None:
            out = torch.empty((n_views, g.n_rows, g.n_cols), dtype=torch.float32, device=vol.device)
        with self._ws_use(self.adjoint_workspace_bytes(n_pitches), stream) as ws:
            self._check(lib().katsevich_adjoint(self._h, _ptr(vol), first_pitch, n_pitches, _ptr(out), sino_first_view,
                                                n_views, _ptr(ws), ws.numel(), _stream_handle(stream)))
        return out

    # -- data generation (NEXT-3) -------------------------------------------
    def project_ellipsoids(self, ellipsoids, first_view: int, n_views: int, out=None, stream=None):
        """Exact line integrals of an ellipsoid phantom [n][8] (host) -> cuda float32 [n_views][rows][cols]."""
        import torch
        e = np.ascontiguousarray(np.asarray(ellipsoids, dtype=np.float64).reshape(-1, 8))
        g = self.geometry
        if out is None:
            out = torch.empty((n_views, g.n_rows, g.n_cols), dtype=torch.float32, device=f"cuda:{self.device}")
        self._check(lib().katsevich_project_ellipsoids(self._h, e.ctypes.data_as(ctypes.c_void_p), e.shape[0],
                                                       first_view, n_views, _ptr(out), _stream_handle(stream)))
        return out

    def project_volume(self, vol, z_first: float, dz: float, first_view: int, n_views: int, out=None, stream=None):
        """Trilinear ray-marched line integrals of vol (cuda float32 [nz][ny][nx]); returns
        (sinogram, number of rays truncated by the volume's z extent)."""
        import torch
        assert vol.is_cuda and vol.dtype == torch.float32 and vol.is_contiguous()
        g = self.geometry
        if out is None:
            out = torch.empty((n_views, g.n_rows, g.n_cols), dtype=torch.float32, device=vol.device)
        nt = ctypes.c_int64()
        self._check(lib().katsevich_project_volume(self._h, _ptr(vol), vol.shape[0], z_first, dz, first_view, n_views,
                                                   _ptr(out), ctypes.byref(nt), _stream_handle(stream)))
        return out, nt.value

    def degrade(self, sino, first_view: int, alpha_stride: int = 4, I0: float = 1e5, gauss_var: float = 0.5,
                seed: int = 0, mode: int = 0, return_counts: bool = False, stream=None):
        """Sparse-view + 'Gaussian+Poisson' degradation (katsevich_degrade) of a cuda float32
        sinogram whose first view is first_view.  Returns out (and counts, M when return_counts)."""
        import torch
        assert sino.is_cuda and sino.dtype == torch.float32 and sino.is_contiguous()
        out = torch.empty_like(sino)
        counts = torch.zeros(sino.shape, dtype=torch.int64, device=sino.device) if return_counts else None
        M = torch.zeros(1, dtype=torch.float32, device=sino.device)
        self._check(lib().katsevich_degrade(self._h, _ptr(sino), first_view, sino.shape[0], alpha_stride, I0,
                                            gauss_var, seed, mode, _ptr(out),
                                            _ptr(counts) if counts is not None else None, _ptr(M),
                                            _stream_handle(stream)))
        return (out, counts, M) if return_counts else out

    def adjoint_batch(self, vols, out=None, stream=None):
        """Transpose of reconstruct_batch (katsevich_adjoint_batch): vols cuda float32
        [B][nz][ny][nx] -> slab adjoints [B][n_slab][rows][cols]."""
        import torch
        assert vols.is_cuda and vols.dtype == torch.float32 and vols.is_contiguous()
        B = vols.shape[0]
        g = self.geometry
        nv = self.pitch_views(0)[1]
        if out is None:
            out = torch.empty((B, nv, g.n_rows, g.n_cols), dtype=torch.float32, device=vols.device)
        b = ctypes.c_size_t()
        self._check(lib().katsevich_adjoint_batch_workspace_bytes(self._h, B, ctypes.byref(b)))
        with self._ws_use(b.value, stream) as ws:
            self._check(lib().katsevich_adjoint_batch(self._h, _ptr(vols), B, _ptr(out), _ptr(ws), ws.numel(),
                                                      _stream_handle(stream)))
        return out

    def filter(self, sino, sino_first_view: int, out_first_view: int, n_out: int, stages=("gF",), stream=None):
        import torch
        g = self.geometry
        npsi = self.table_info()["n_psi"]
        dev = sino.device
        nr_f, nc_f = self.filtered_grid()
        gF = torch.empty((n_out, nr_f, nc_f), dtype=torch.float32, device=dev)
        g3 = torch.empty((n_out, npsi, nc_f), dtype=torch.float32, device=dev) if "g3" in stages else None
        g4 = torch.empty((n_out, npsi, nc_f), dtype=torch.float32, device=dev) if "g4" in stages else None
        self._check(lib().katsevich_filter(self._h, _ptr(sino), sino_first_view, sino.shape[0], out_first_view, n_out,
                                           _ptr(g3) if g3 is not None else None,
                                           _ptr(g4) if g4 is not None else None, _ptr(gF), _stream_handle(stream)))
        return {"g3": g3, "g4": g4, "gF": gF}

    def backproject(self, gF, gF_first_view: int, pitch: int = 0, out=None, stream=None):
        import torch
        if out is None:
            out = torch.empty(self._vol_shape(1), dtype=torch.float32, device=gF.device)
        self._check(lib().katsevich_backproject(self._h, _ptr(gF), gF_first_view, gF.shape[0], pitch, _ptr(out),
                                                _stream_handle(stream)))
        return out

    BP_KERNELS = {0: None, 1: "k_backproject", 2: "k_bp_window", 3: "k_bp_tmem", 4: "k_bp_items"}

    def bp_kernel(self):
        """Name of the step-7 kernel variant the last backprojection launched
        (katsevich_bp_kernel), or None before the first one."""
        r = lib().katsevich_bp_kernel(self._h)
        if r < 0:
            self._check(r)
        return self.BP_KERNELS[r]

    # -- in-run timing -------------------------------------------------------
    def profile_enable(self, enable: bool = True):
        self._check(lib().katsevich_profile_enable(self._h, 1 if enable else 0))

    def profile_read(self, reset: bool = True):
        st = KatsevichStats()
        self._check(lib().katsevich_profile_read(self._h, ctypes.byref(st), 1 if reset else 0))
        return {"launches": {STAGES[i]: st.launches[i] for i in range(6)},
                "ms": {STAGES[i]: st.ms[i] for i in range(6)},
                "busy_ms": {STAGES[i]: st.busy_ms[i] for i in range(6)},
                "total_launches": st.total_launches}
