"""Python handle of a device plan (``kfbi_plan`` of the C ABI).

A plan owns the per-grid device tables (twiddles, eigenvalue table), the
panel scratch of the box solver and, once ``set_geometry`` ran, the uploaded
geometry tables of one InterfaceWorkspace.  All field arguments are torch
CUDA tensors; work is enqueued on the backend's current stream.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N

_F64 = np.float64
_BOX = {"dirichlet-zero": 0, "neumann-zero": 1}
_KIND = {"dirichlet": 0, "neumann": 1}


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _addr(x):
    """Device address of a tensor or a raw integer pointer."""
    return int(x) if isinstance(x, int) else x.data_ptr()


def _ptr_table(bufs):
    """C array of device addresses (tensors or raw integer pointers)."""
    return (C.c_void_p * len(bufs))(*[_addr(b) for b in bufs])


class Plan:
    def __init__(self, m, h, backend):
        self.m = int(m)
        self.h = float(h)
        self.backend = backend
        self.device = backend.device
        self._lib = N.lib()
        desc = N.GridDesc(self.m, self.h, self.device)
        handle = C.c_void_p()
        N.check(self._lib.kfbi_plan_create(C.byref(desc), C.byref(handle)))
        self.handle = handle
        self.has_geometry = False
        self.has_onesided = False
        self._keep = []
        backend.register(self)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._lib.kfbi_plan_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self.handle = None

    # -- accounting ---------------------------------------------------------
    def set_timing(self, enabled):
        N.check(self._lib.kfbi_set_timing(self.handle, int(bool(enabled))))

    def kernel_times(self):
        ms = (C.c_double * 9)()
        calls = (C.c_int64 * 9)()
        N.check(self._lib.kfbi_kernel_times(self.handle, ms, calls))
        return ({k: ms[i] for i, k in enumerate(N.KERNEL_ORDER)},
                {k: calls[i] for i, k in enumerate(N.KERNEL_ORDER)})

    def reset_kernel_times(self):
        N.check(self._lib.kfbi_reset_kernel_times(self.handle))

    def launch_count(self):
        return int(self._lib.kfbi_launch_count(self.handle))

    @property
    def stream(self):
        return self.backend.stream_handle()

    # -- geometry -----------------------------------------------------------
    def set_geometry(self, tables):
        """Upload the host tables built by InterfaceWorkspace (dict of numpy)."""
        t = {
            "edge_axis": _c(tables["edge_axis"], np.int8),
            "rec_edge": _c(tables["rec_edge"], np.int32),
            "rec_d": _c(tables["rec_d"], _F64),
            "rec_sigma": _c(tables["rec_sigma"], _F64),
            "group_start": _c(tables["group_start"], np.int32),
            "group_node": _c(tables["group_node"], np.int32),
            "row_group": _c(tables["row_group"], np.int32),
            "deriv_col": _c(tables["deriv_col"], _F64),
            "speed": _c(tables["speed"], _F64),
            "tangent": _c(tables["tangent"], _F64),
            "normal": _c(tables["normal"], _F64),
            "dtan_ds": _c(tables["dtan_ds"], _F64),
            "inv3": _c(tables["inv3"], _F64),
            "stencil": _c(tables["stencil"], np.int32),
            "ainv_rows": _c(tables["ainv_rows"], _F64),
            "jcoef": _c(tables["jcoef"], _F64),
        }
        # W: host rows when given, else built on the device from the crossing
        # and control parameters (trigonometric interpolation)
        if tables.get("w_edges") is not None:
            t["w_edges"] = _c(tables["w_edges"], _F64)
        else:
            t["edge_theta"] = _c(tables["edge_theta"], _F64)
            t["ctl_theta"] = _c(tables["ctl_theta"], _F64)
        g = N.Geometry(
            n_ctl=int(tables["n_ctl"]), n_edges=int(t["edge_axis"].size),
            n_rec=int(t["rec_edge"].size), n_groups=int(t["group_node"].size),
            **{k: v.ctypes.data for k, v in t.items()})
        N.check(self._lib.kfbi_plan_set_geometry(self.handle, C.byref(g)))
        self.n_ctl = int(tables["n_ctl"])
        self.n_edges = int(t["edge_axis"].size)
        self.has_geometry = True

    def set_interp(self, mode):
        """Edge-value form: "auto" (spectral when it applies), "w" (W rows),
        "spectral" (kfbi_plan_set_interp)."""
        N.check(self._lib.kfbi_plan_set_interp(self.handle, {"auto": 0, "w": 1, "spectral": 2}[mode]))

    _COLS = ("auto", "tridiagonal", "dst")

    def set_colsolver(self, mode):
        """Column stage of the dirichlet box solve: "auto" (default: the
        tridiagonal recurrences when they agree with the reference's DST
        route to <= 1e-11, see kfbi_plan_set_colsolver), "tridiagonal"
        (factored recurrences) or "dst" (DST-I -> divide -> DST-I)."""
        N.check(self._lib.kfbi_plan_set_colsolver(self.handle, self._COLS.index(mode)))

    def set_facr(self, on):
        """Cyclic-reduction (FACR(1)) form of the dirichlet box solve
        (kfbi_plan_set_facr, default on where it applies)."""
        N.check(self._lib.kfbi_plan_set_facr(self.handle, int(bool(on))))

    def facr_for(self, kappa):
        """True when a single-slab dirichlet box solve with kappa uses FACR(1)."""
        kappa = complex(kappa)
        v = C.c_int32(0)
        N.check(self._lib.kfbi_plan_facr_for(self.handle, kappa.real, kappa.imag, C.byref(v)))
        return bool(v.value)

    def set_trace_sweep(self, on):
        """Operator form, Dirichlet: sweep 1 forms only its trace (stencil
        nodes) instead of the whole field (kfbi_plan_set_trace_sweep)."""
        N.check(self._lib.kfbi_plan_set_trace_sweep(self.handle, int(bool(on))))

    @property
    def colsolver(self):
        v = C.c_int32(0)
        N.check(self._lib.kfbi_plan_get_colsolver(self.handle, C.byref(v)))
        return self._COLS[v.value]

    def colsolver_for(self, kappa):
        """("tridiagonal" | "dst", deviation bound E) chosen for this kappa."""
        kappa = complex(kappa)
        t, e = C.c_int32(0), C.c_double(0.0)
        N.check(self._lib.kfbi_plan_colsolver_for(self.handle, kappa.real, kappa.imag,
                                                  C.byref(t), C.byref(e)))
        return ("tridiagonal" if t.value else "dst"), float(e.value)

    @property
    def operator_max_controls(self):
        """Largest n_ctl the on-chip operator sweeps support on this device
        (kfbi_operator_max_controls)."""
        v = C.c_int32(0)
        N.check(self._lib.kfbi_operator_max_controls(self.handle, C.byref(v)))
        return int(v.value)

    @property
    def spectral_edges(self):
        v = C.c_int32(0)
        N.check(self._lib.kfbi_plan_get_interp(self.handle, C.byref(v)))
        return bool(v.value)

    def copy_w(self, row0, nrows):
        """Rows of the device W (setup check)."""
        out = np.empty((int(nrows), self.n_ctl))
        N.check(self._lib.kfbi_plan_copy_w(self.handle, int(row0), int(nrows), out.ctypes.data))
        return out

    # -- kernels --------------------------------------------------------------
    @staticmethod
    def _dt(cplx):
        return N.C128 if cplx else N.F64

    def box_solve(self, rhs, u, kappa, bc="dirichlet-zero"):
        k = complex(kappa)
        N.check(self._lib.kfbi_box_solve_bc(self.handle, self._dt(u.is_complex()), _BOX[bc],
                                            k.real, k.imag, rhs.data_ptr(), u.data_ptr(),
                                            self.stream))

    # -- slab-decomposed box solve (dist.py) ----------------------------------
    def slab_panel_bytes(self, cplx, nranks):
        b = C.c_int64(0)
        N.check(self._lib.kfbi_slab_panel_bytes(self.handle, self._dt(cplx), int(nranks), C.byref(b)))
        return b.value

    def slab_rows_fwd(self, cplx, nranks, rank, rhs, panels, sign=1.0, jv=None):
        sl = N.Slab(int(nranks), int(rank))
        N.check(self._lib.kfbi_slab_rows_fwd(self.handle, self._dt(cplx), C.byref(sl), N.ptr(rhs),
                                             float(sign), N.ptr(jv), panels.data_ptr(), self.stream))

    def slab_cols(self, cplx, nranks, rank, kappa, panels):
        k = complex(kappa)
        sl = N.Slab(int(nranks), int(rank))
        N.check(self._lib.kfbi_slab_cols(self.handle, self._dt(cplx), C.byref(sl), k.real, k.imag,
                                         panels.data_ptr(), self.stream))

    def slab_rows_inv(self, cplx, nranks, rank, panels, u):
        sl = N.Slab(int(nranks), int(rank))
        N.check(self._lib.kfbi_slab_rows_inv(self.handle, self._dt(cplx), C.byref(sl),
                                             _addr(panels), u.data_ptr(), self.stream))

    def slab_rows_fwd_p2p(self, cplx, nranks, rank, rhs, peers, sign=1.0, jv=None):
        """Forward row pass storing panel chunk h into peers[h] (rank h's
        column-pass buffer): the first all-to-all fused into the stores."""
        sl = N.Slab(int(nranks), int(rank))
        tab = _ptr_table(peers)
        N.check(self._lib.kfbi_slab_rows_fwd_p2p(self.handle, self._dt(cplx), C.byref(sl),
                                                 N.ptr(rhs), float(sign), N.ptr(jv), tab,
                                                 self.stream))

    def slab_cols_p2p(self, cplx, nranks, rank, kappa, panels, peers):
        """Column pass on the own buffer, storing row chunk h into peers[h]
        (rank h's row-pass buffer): the second all-to-all fused."""
        k = complex(kappa)
        sl = N.Slab(int(nranks), int(rank))
        tab = _ptr_table(peers)
        N.check(self._lib.kfbi_slab_cols_p2p(self.handle, self._dt(cplx), C.byref(sl), k.real,
                                             k.imag, _addr(panels), tab, self.stream))

    def slab_tri_bytes(self, cplx, nranks):
        a, f = C.c_int64(0), C.c_int64(0)
        N.check(self._lib.kfbi_slab_tri_bytes(self.handle, self._dt(cplx), int(nranks), C.byref(a),
                                              C.byref(f)))
        return a.value, f.value

    def slab_cols_tri(self, cplx, nranks, rank, kappa, panels, agg, flags, epoch, timed_out=None,
                      max_spins=1 << 26, virt_panels=None):
        """Transpose-free column stage (kfbi_slab_cols_tri): agg / flags are
        every rank's buffers as mapped here; virt_panels: all ranks in one
        launch on this device."""
        k = complex(kappa)
        d = N.TriDist(nranks=int(nranks), rank=int(rank), virt=int(virt_panels is not None),
                      epoch=int(epoch), max_spins=int(max_spins),
                      timed_out=N.ptr(timed_out) if timed_out is not None else None)
        for h in range(int(nranks)):
            d.agg[h] = _addr(agg[h])
            d.flags[h] = _addr(flags[h])
            if virt_panels is not None:
                d.panels[h] = _addr(virt_panels[h])
        N.check(self._lib.kfbi_slab_cols_tri(self.handle, self._dt(cplx), int(nranks), int(rank),
                                             k.real, k.imag, _addr(panels) if panels is not None else None,
                                             C.byref(d), self.stream))

    def p2p_barrier(self, flags, nranks, rank, epoch, timed_out=None, max_spins=0):
        tab = _ptr_table(flags)
        N.check(self._lib.kfbi_p2p_barrier(tab, int(nranks), int(rank), int(epoch),
                                           int(max_spins), N.ptr(timed_out), self.stream))

    # -- slab-decomposed Richardson sweep (dist.py) -------------------------------
    def edge_values(self, jm, jv):
        N.check(self._lib.kfbi_edge_values(self.handle, self._dt(jm.is_complex()), jm.data_ptr(),
                                           jv.data_ptr(), self.stream))

    def slab_stencil_values(self, bc_kind, nranks, rank, u_slab, vals):
        sl = N.Slab(int(nranks), int(rank))
        N.check(self._lib.kfbi_slab_stencil_values(self.handle, self._dt(vals.is_complex()),
                                                   _KIND[bc_kind], C.byref(sl), u_slab.data_ptr(),
                                                   vals.data_ptr(), self.stream))

    def rich_begin(self, max_iter, tol):
        N.check(self._lib.kfbi_rich_begin(self.handle, int(max_iter), float(tol), self.stream))

    def slab_update(self, bc_kind, vals, jm, g, density, trace_u, trace_un, gamma):
        N.check(self._lib.kfbi_slab_update(self.handle, self._dt(vals.is_complex()), _KIND[bc_kind],
                                           vals.data_ptr(), jm.data_ptr(), g.data_ptr(),
                                           density.data_ptr(), trace_u.data_ptr(),
                                           trace_un.data_ptr(), float(gamma), self.stream))

    def rich_state(self, max_iter):
        it, done, res = C.c_int32(0), C.c_int32(0), C.c_double(0.0)
        hist = np.zeros(max(int(max_iter), 1))
        N.check(self._lib.kfbi_rich_state(self.handle, C.byref(it), C.byref(done), C.byref(res),
                                          hist.ctypes.data, self.stream))
        return it.value, done.value, res.value, hist[: it.value].tolist()

    def jumps(self, kappa, phi, psi, f_gamma, jm, f_gamma_sign=1.0):
        k = complex(kappa)
        N.check(self._lib.kfbi_jumps(self.handle, self._dt(jm.is_complex()), k.real, k.imag,
                                     N.ptr(phi), N.ptr(psi), f_gamma.data_ptr(),
                                     float(f_gamma_sign), jm.data_ptr(), self.stream))

    def corrections(self, jm, c):
        N.check(self._lib.kfbi_corrections(self.handle, self._dt(jm.is_complex()), jm.data_ptr(),
                                           c.data_ptr(), self.stream))

    def interface_solve(self, kappa, F, jm, u, bc="dirichlet-zero"):
        k = complex(kappa)
        N.check(self._lib.kfbi_interface_solve_bc(self.handle, self._dt(u.is_complex()), _BOX[bc],
                                                  k.real, k.imag, F.data_ptr(), jm.data_ptr(),
                                                  u.data_ptr(), self.stream))

    def extract(self, u, jm, out):
        N.check(self._lib.kfbi_extract(self.handle, self._dt(out.is_complex()), u.data_ptr(),
                                       jm.data_ptr(), out.data_ptr(), self.stream))

    def set_onesided(self, stencil7, rows, fallback_mask):
        """Upload the OneSidedExtractor tables (Neumann BVPs)."""
        st = _c(stencil7, np.int32)
        rw = _c(rows, _F64)
        fb = _c(fallback_mask, np.uint8)
        N.check(self._lib.kfbi_plan_set_onesided(self.handle, int(st.shape[0]),
                                                 st.ctypes.data, rw.ctypes.data, fb.ctypes.data))
        self.has_onesided = True

    def extract_onesided(self, u, jm, out):
        N.check(self._lib.kfbi_extract_onesided(self.handle, self._dt(out.is_complex()),
                                                u.data_ptr(), jm.data_ptr(), out.data_ptr(),
                                                self.stream))

    def build_operator(self, kappa, cplx, bc_kind="dirichlet", box_bc=None):
        """Trace operator T of this geometry for one kappa and BVP kind (n_ctl
        pipeline evaluations, once per (geometry, kappa, kind))."""
        k = complex(kappa)
        box_bc = box_bc or ("dirichlet-zero" if bc_kind == "dirichlet" else "neumann-zero")
        N.check(self._lib.kfbi_build_trace_operator_bc(
            self.handle, self._dt(cplx), _KIND[bc_kind], _BOX[box_bc], k.real, k.imag,
            self.stream))
        self.operator_key = (k, bool(cplx), bc_kind, box_bc)

    def richardson(self, *, kappa, F, F_sign, f_gamma, f_gamma_sign, g, density, gamma, tol,
                   max_iter, u, trace_u, trace_un, sweeps_hint=0, use_operator=False,
                   log_slot=-1, bc_kind="dirichlet", box_bc=None, field_chunks=False):
        k = complex(kappa)
        box_bc = box_bc or ("dirichlet-zero" if bc_kind == "dirichlet" else "neumann-zero")
        b = N.Bvp(dtype=self._dt(u.is_complex()), kappa_re=k.real, kappa_im=k.imag,
                  F=F.data_ptr(), F_sign=float(F_sign), f_gamma=f_gamma.data_ptr(),
                  f_gamma_sign=float(f_gamma_sign), g=g.data_ptr(), density=density.data_ptr(),
                  gamma=float(gamma), tol=float(tol), max_iter=int(max_iter),
                  sweeps_hint=int(sweeps_hint), u=u.data_ptr(), trace_u=trace_u.data_ptr(),
                  trace_un=trace_un.data_ptr(), use_operator=int(bool(use_operator)),
                  log_slot=int(log_slot), bc_kind=_KIND[bc_kind], box_bc=_BOX[box_bc],
                  field_chunks=int(bool(field_chunks)))
        hist = np.zeros(max(int(max_iter), 1))
        res = N.BvpResult(history=hist.ctypes.data_as(C.POINTER(C.c_double)))
        status = self._lib.kfbi_richardson(self.handle, C.byref(b), C.byref(res), self.stream)
        if log_slot >= 0:                       # asynchronous: results pending in the log
            N.check(status)
            return None, None, None
        history = hist[: res.iterations].tolist()
        last = history[-1] if history else None
        N.check(status, iterations=int(max_iter), last_residual=last)
        return res.iterations, res.residual, history

    def gmres(self, *, kappa, F, F_sign, f_gamma, f_gamma_sign, g, density, gamma, tol, max_iter,
              u, trace_u, trace_un, restart=40, use_operator=False, bc_kind="dirichlet",
              box_bc=None):
        """Opt-in restarted GMRES on the same BIE (kfbi_gmres); density in place."""
        k = complex(kappa)
        box_bc = box_bc or ("dirichlet-zero" if bc_kind == "dirichlet" else "neumann-zero")
        b = N.Bvp(dtype=self._dt(u.is_complex()), kappa_re=k.real, kappa_im=k.imag,
                  F=F.data_ptr(), F_sign=float(F_sign), f_gamma=f_gamma.data_ptr(),
                  f_gamma_sign=float(f_gamma_sign), g=g.data_ptr(), density=density.data_ptr(),
                  gamma=float(gamma), tol=float(tol), max_iter=int(max_iter), sweeps_hint=0,
                  u=u.data_ptr(), trace_u=trace_u.data_ptr(), trace_un=trace_un.data_ptr(),
                  use_operator=int(bool(use_operator)), log_slot=-1, bc_kind=_KIND[bc_kind],
                  box_bc=_BOX[box_bc])
        hist = np.zeros(max(int(max_iter), 1))
        res = N.BvpResult(history=hist.ctypes.data_as(C.POINTER(C.c_double)))
        status = self._lib.kfbi_gmres(self.handle, C.byref(b), int(restart), C.byref(res),
                                      self.stream)
        n_hist = max(0, min(int(max_iter), res.iterations))
        history = [h for h in hist[:n_hist].tolist()]
        N.check(status, iterations=int(max_iter), last_residual=res.residual)
        return res.iterations, res.residual, history

    # -- asynchronous step log ----------------------------------------------
    def log_reserve(self, count):
        N.check(self._lib.kfbi_log_reserve(self.handle, int(count)))

    def log_norm(self, slot, which=0):
        N.check(self._lib.kfbi_log_norm(self.handle, int(slot), int(which), self.stream))

    def set_exterior_zero(self, on):
        """The masked outputs of the right-hand-side kernels are zero outside
        the mask already (kfbi_plan_set_exterior_zero)."""
        N.check(self._lib.kfbi_plan_set_exterior_zero(self.handle, int(bool(on))))

    def set_field_chunks(self, pairs):
        """(odd row, 16-node chunk) pairs covering the nodes a caller reads
        of fields returned with field_chunks=True (kfbi_plan_set_field_chunks)."""
        arr = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 2)
        N.check(self._lib.kfbi_plan_set_field_chunks(self.handle, arr.ctypes.data, int(arr.shape[0])))

    def work_fractions(self):
        """(even rows trace, even rows field, odd chunks trace, odd chunks
        field) fractions of the reduced FACR solves (kfbi_plan_work_fractions)."""
        out = (C.c_double * 4)()
        N.check(self._lib.kfbi_plan_work_fractions(self.handle, out))
        return tuple(out)

    def set_interior_list(self, idx):
        """Interior node list (device int32 tensor, kept alive by the
        caller) for the masked Newton passes; None clears it."""
        if idx is None:
            N.check(self._lib.kfbi_plan_set_interior_list(self.handle, None, 0))
        else:
            N.check(self._lib.kfbi_plan_set_interior_list(self.handle, idx.data_ptr(), int(idx.numel())))

    def log_clear(self, slot, count=1):
        N.check(self._lib.kfbi_log_clear(self.handle, int(slot), int(count), self.stream))

    def log_copy(self, src, dst, count=1):
        N.check(self._lib.kfbi_log_copy(self.handle, int(src), int(dst), int(count), self.stream))

    def log_fetch(self, first, count):
        out = (N.StepLog * max(int(count), 1))()
        N.check(self._lib.kfbi_log_fetch(self.handle, int(first), int(count), out, self.stream))
        return [(out[i].iterations, out[i].status, out[i].residual, out[i].norm, out[i].newton)
                for i in range(int(count))]

    def heat_rhs(self, n, mask, u, F_old, F_new, a, want_norm=True):
        norm = C.c_double(0.0)
        N.check(self._lib.kfbi_heat_rhs(self.handle, int(n), N.ptr(mask), u.data_ptr(),
                                        F_old.data_ptr(), F_new.data_ptr(), float(a),
                                        C.byref(norm) if want_norm else None, self.stream))
        return norm.value

    def wave_rhs(self, n, mask, u_next, u_curr, F_curr, F_prev, F_new, kw, coef, want_norm=True):
        norm = C.c_double(0.0)
        N.check(self._lib.kfbi_wave_rhs(self.handle, int(n), N.ptr(mask), u_next.data_ptr(),
                                        u_curr.data_ptr(), F_curr.data_ptr(), F_prev.data_ptr(),
                                        F_new.data_ptr(), float(kw), float(coef),
                                        C.byref(norm) if want_norm else None, self.stream))
        return norm.value

    def schr_ustar(self, n, mode, u, other, tau, out):
        N.check(self._lib.kfbi_schr_ustar(self.handle, int(n), int(mode), u.data_ptr(),
                                          other.data_ptr(), float(tau), out.data_ptr(),
                                          self.stream))

    def nonlinear_phase(self, n, ustar, v, w, half_tau, mask, out, kappa=None, F=None,
                        log_slot=None):
        k = complex(kappa) if kappa is not None else 0j
        res = C.c_double(0.0)
        status = self._lib.kfbi_nonlinear_phase(
            self.handle, int(n), ustar.data_ptr(), v.data_ptr(), float(w), float(half_tau),
            N.ptr(mask), out.data_ptr(), k.real, k.imag, N.ptr(F),
            None if log_slot is not None else C.byref(res), self.stream)
        if log_slot is not None:
            N.check(status)
            self.log_norm(log_slot, which=1)
            return None
        N.check(status, iterations=50, last_residual=res.value)
        return res.value

    def strang_phase(self, n, mode, u, other, tau, v, w, half_tau, mask, out, kappa=None,
                     F=None, log_slot=None):
        """schr_ustar + nonlinear_phase in one pass (kfbi_strang_phase)."""
        k = complex(kappa) if kappa is not None else 0j
        res = C.c_double(0.0)
        status = self._lib.kfbi_strang_phase(
            self.handle, int(n), int(mode), u.data_ptr(), other.data_ptr(), float(tau),
            v.data_ptr(), float(w), float(half_tau), N.ptr(mask), out.data_ptr(), k.real, k.imag,
            N.ptr(F), None if log_slot is not None else C.byref(res), self.stream)
        if log_slot is not None:
            N.check(status)
            self.log_norm(log_slot, which=1)
            return None
        N.check(status, iterations=50, last_residual=res.value)
        return res.value

    def gather(self, idx, src, dst):
        """dst[i] = src[idx[i]] on the device (kfbi_gather)."""
        N.check(self._lib.kfbi_gather(self.handle, self._dt(src.is_complex()), int(idx.numel()),
                                      idx.data_ptr(), src.data_ptr(), dst.data_ptr(), self.stream))

    def mask_norm(self, n, mask, u, want_norm=True):
        norm = C.c_double(0.0)
        N.check(self._lib.kfbi_mask_norm(self.handle, self._dt(u.is_complex()), int(n),
                                         N.ptr(mask), u.data_ptr(),
                                         C.byref(norm) if want_norm else None, self.stream))
        return norm.value
