"""Python binding of the sgm C ABI (include/sgm.h) -- argument marshalling only.

Every computation runs in the CUDA kernels of ``libsgm.so`` (sm_100a).  There is no CPU
fallback: importing this package without the built library raises, and device calls on a
machine without a GPU fail with the library's status code.

Low-level: the C functions are exposed with their C names (``sgm_plan_create``, ``sgm_step``,
...) taking plain integers for pointers.  High-level: :class:`Plan` accepts torch CUDA float64
tensors and passes ``tensor.data_ptr()`` and ``torch.cuda.current_stream().cuda_stream``.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SGM_LIB_VARIANT=checked selects the verification build libsgm_checked.so (build.py checked=True:
# run-time protocol checks of the pipelined sweeps, csrc/check.cuh); the default is the product
# library.  The variant is chosen once, at import.
VARIANT = os.environ.get("SGM_LIB_VARIANT", "")
if VARIANT not in ("", "checked"):
    raise ImportError(f"SGM_LIB_VARIANT={VARIANT!r}: only 'checked' is known")
LIB_PATH = os.path.join(_HERE, "libsgm_checked.so" if VARIANT == "checked" else "libsgm.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2302_04979_b200.build` "
                      "(nvcc, sm_100a); there is no fallback path")

_lib = ctypes.CDLL(LIB_PATH)

c_int, c_double, c_size_t, c_void_p = ctypes.c_int, ctypes.c_double, ctypes.c_size_t, ctypes.c_void_p
c_dp = ctypes.POINTER(ctypes.c_double)


class sgm_lifting(ctypes.Structure):
    """Time-separable inhomogeneous Dirichlet data (sgm.h, sgm_step_lifted): device pointers."""
    _fields_ = [("w_e", c_void_p), ("c_b", c_void_p), ("q0", c_void_p), ("q1", c_void_p), ("g", c_void_p),
                ("beta", c_void_p)]


class sgm_plan_desc(ctypes.Structure):
    _fields_ = [("n_el", c_int * 3), ("degree", c_int), ("geom_ctrl", c_void_p),
                ("quad_points", c_int), ("device", c_int), ("geom_weights", c_void_p)]


STATUS = {0: "SGM_OK", 1: "SGM_E_INVALID_ARG", 2: "SGM_E_UNSUPPORTED", 3: "SGM_E_GEOMETRY",
          4: "SGM_E_MATERIAL", 5: "SGM_E_SINGULAR", 6: "SGM_E_SOURCE_DIVERGENCE", 7: "SGM_E_CUDA",
          8: "SGM_E_NOMEM"}
FORM_E, FORM_D, FORM_B, FORM_H = 0, 1, 2, 3
K1, KT1 = 0, 1
MASS_EPS, MASS_MU = 0, 1
CURL_PRIMAL, CURL_DUAL = 0, 1
EPS, MU = 0, 1
K_CLASSES = ["eps_z", "eps_y", "eps_x", "mu_z", "mu_y", "mu_x", "update", "hodge_general", "solve_z",
             "fused_eps", "fused_mu"]
# schedule options (sgm.h SGM_OPT_*)
OPT_FULL_SCHEDULE, OPT_EXACT_SPIKE, OPT_SERIAL, OPT_NO_GRAPH, OPT_FUSED, OPT_WIDE_TILES = 0x1, 0x2, 0x4, 0x8, 0x10, 0x20
OPT_OTF_GEOMETRY = 0x40
TAB_G, TAB_M, TAB_GAMMA_B1, TAB_GAMMA_C2, TAB_GAMMA_BP, TAB_GAMMA_C1 = range(6)

_SIGS = {
    "sgm_plan_create": [ctypes.POINTER(sgm_plan_desc), ctypes.POINTER(c_void_p)],
    "sgm_plan_destroy": [c_void_p],
    "sgm_plan_len": [c_void_p, c_int, ctypes.POINTER(c_size_t)],
    "sgm_plan_shape": [c_void_p, c_int, c_int, ctypes.POINTER(c_int)],
    "sgm_plan_qp_count": [c_void_p, ctypes.POINTER(c_size_t)],
    "sgm_plan_qp_coords": [c_void_p, c_void_p],
    "sgm_plan_table": [c_void_p, c_int, c_int, c_void_p, ctypes.POINTER(c_int)],
    "sgm_plan_hodge_separable": [c_void_p, c_int, ctypes.POINTER(c_int)],
    "sgm_plan_set_material": [c_void_p, c_int, c_void_p, c_double],
    "sgm_workspace_bytes": [c_void_p, ctypes.POINTER(c_size_t)],
    "sgm_step": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_int,
                 c_void_p, c_size_t, c_void_p],
    "sgm_step_lifted": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_double,
                        c_int, c_void_p, c_size_t, c_void_p],
    "sgm_step_eh": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_int, c_void_p, c_size_t, c_void_p],
    "sgm_step_host": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_int,
                      c_void_p],
    "sgm_step_composed": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int,
                          c_double, c_int, c_void_p, c_size_t, c_void_p],
    "sgm_kron_solve": [c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p],
    "sgm_pairing_apply": [c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p],
    "sgm_hodge_apply": [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p],
    "sgm_hodge_star": [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p],
    "sgm_curl": [c_void_p, c_int, c_void_p, c_void_p, c_void_p],
    "sgm_energy": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p],
    "sgm_gauss": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p],
    "sgm_cfl": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_size_t, c_void_p],
    "sgm_check_source": [c_void_p, c_void_p, c_void_p, c_size_t, c_void_p],
    "sgm_plan_kernels_per_step": [c_void_p, ctypes.POINTER(c_int)],
    "sgm_plan_reduced_schedule": [c_void_p, ctypes.POINTER(c_int)],
    "sgm_plan_set_scheme": [c_void_p, c_int],
    "sgm_plan_set_options": [c_void_p, ctypes.c_uint],
    "sgm_plan_get_options": [c_void_p, ctypes.POINTER(ctypes.c_uint)],
    "sgm_geometry_greville": [c_int, c_int, c_void_p],
    "sgm_geometry_interpolate": [c_void_p, c_int, c_void_p, c_void_p],
    "sgm_plan_set_profiling": [c_void_p, c_int],
    "sgm_plan_profile": [c_void_p, c_void_p, c_void_p],
    "sgm_check_read": [c_int, ctypes.POINTER(ctypes.c_uint), ctypes.POINTER(ctypes.c_uint)],
}
for _name, _args in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = c_int
    globals()[_name] = _f
_lib.sgm_last_error.restype = ctypes.c_char_p
_lib.sgm_last_error.argtypes = []
_lib.sgm_version.restype = ctypes.c_char_p
_lib.sgm_version.argtypes = []
sgm_last_error = _lib.sgm_last_error
sgm_version = _lib.sgm_version

EXPORTED = list(_SIGS) + ["sgm_last_error", "sgm_version"]


class SgmError(RuntimeError):
    def __init__(self, status, where):
        self.status = status
        super().__init__(f"{where}: {STATUS.get(status, status)}: {sgm_last_error().decode()}")


def check(status, where="sgm"):
    if status != 0:
        raise SgmError(status, where)


def check_read(reset=True):
    """Verification build only (SGM_LIB_VARIANT=checked): (violations, first code) of the sweep
    protocol checks since the last reset (sgm.h sgm_check_read); the product build raises."""
    n, f = ctypes.c_uint(0), ctypes.c_uint(0)
    check(sgm_check_read(1 if reset else 0, ctypes.byref(n), ctypes.byref(f)), "sgm_check_read")
    return n.value, f.value


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, int):
        return t
    if hasattr(t, "data_ptr"):
        import torch
        if t.dtype != torch.float64 or not t.is_contiguous():
            raise ValueError("tensors must be contiguous float64")
        return t.data_ptr()
    raise TypeError(type(t))


def _stream(stream):
    if stream is not None:
        return stream if isinstance(stream, int) else stream.cuda_stream
    import torch
    return torch.cuda.current_stream().cuda_stream


def interpolate_geometry(n_el, degree, fmap):
    """Control points of a map F: X[..., 3] -> F[..., 3] interpolated in S_p(Xi)^3 at the Greville
    points (sgm_geometry_greville / sgm_geometry_interpolate)."""
    n = (n_el,) * 3 if np.isscalar(n_el) else tuple(n_el)
    gs = []
    for a in range(3):
        g = np.empty(n[a] + degree)
        check(sgm_geometry_greville(n[a], degree, g.ctypes.data), "sgm_geometry_greville")
        gs.append(g)
    Z, Y, X = np.meshgrid(gs[2], gs[1], gs[0], indexing="ij")
    vals = np.ascontiguousarray(fmap(np.stack([X, Y, Z], -1)), dtype=np.float64)
    ctrl = np.empty_like(vals)
    nn = (c_int * 3)(*n)
    check(sgm_geometry_interpolate(nn, degree, vals.ctypes.data, ctrl.ctypes.data), "sgm_geometry_interpolate")
    return ctrl


# Yoshida's 4th-order symmetric composition ("triple jump") of leapfrog sub-steps
_CBRT2 = 2.0 ** (1.0 / 3.0)
YOSHIDA4 = (1.0 / (2.0 - _CBRT2), -_CBRT2 / (2.0 - _CBRT2), 1.0 / (2.0 - _CBRT2))


class Plan:
    """Owning wrapper of an ``sgm_plan`` (marshalling only)."""

    def __init__(self, n_el, degree, geom_ctrl=None, quad_points=0, device=0, geom_weights=None):
        """geom_ctrl: control points [(nz+p)][(ny+p)][(nx+p)][3], or any object with arrays .P (points)
        and .w (weights) describing a rational map; geom_weights: weights of a rational map."""
        n = (n_el,) * 3 if np.isscalar(n_el) else tuple(n_el)
        self.n_el, self.p, self.device = n, degree, device
        if geom_ctrl is not None and hasattr(geom_ctrl, "P") and hasattr(geom_ctrl, "w"):
            geom_ctrl, geom_weights = geom_ctrl.P, geom_ctrl.w
        self._ctrl = None if geom_ctrl is None else np.ascontiguousarray(geom_ctrl, dtype=np.float64)
        self._wts = None if geom_weights is None else np.ascontiguousarray(geom_weights, dtype=np.float64)
        self.geom = geom_ctrl is not None
        desc = sgm_plan_desc((c_int * 3)(*n), degree,
                             None if self._ctrl is None else self._ctrl.ctypes.data, quad_points, device,
                             None if self._wts is None else self._wts.ctypes.data)
        h = c_void_p()
        check(sgm_plan_create(ctypes.byref(desc), ctypes.byref(h)), "sgm_plan_create")
        self.h = h.value
        self._ws = None

    def close(self):
        if getattr(self, "h", None):
            sgm_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --- queries ---
    def len(self, form):
        n = c_size_t()
        check(sgm_plan_len(self.h, form, ctypes.byref(n)), "sgm_plan_len")
        return n.value

    @property
    def N_e(self):
        return self.len(FORM_E)

    @property
    def N_h(self):
        return self.len(FORM_H)

    def shape(self, form, comp):
        xyz = (c_int * 3)()
        check(sgm_plan_shape(self.h, form, comp, xyz), "sgm_plan_shape")
        return tuple(xyz)

    def qp_count(self):
        n = c_size_t()
        check(sgm_plan_qp_count(self.h, ctypes.byref(n)))
        return n.value

    def qp_coords(self):
        out = np.empty((self.qp_count(), 3))
        check(sgm_plan_qp_coords(self.h, out.ctypes.data), "sgm_plan_qp_coords")
        return out

    def table(self, which, axis):
        L = c_int()
        check(sgm_plan_table(self.h, which, axis, None, ctypes.byref(L)))
        out = np.empty((L.value, L.value))
        check(sgm_plan_table(self.h, which, axis, out.ctypes.data, ctypes.byref(L)), "sgm_plan_table")
        return out

    def separable(self, mass):
        s = c_int()
        check(sgm_plan_hodge_separable(self.h, mass, ctypes.byref(s)))
        return bool(s.value)

    def set_material(self, which, values=None, c=1.0):
        if values is None:
            check(sgm_plan_set_material(self.h, which, None, float(c)), "sgm_plan_set_material")
        else:
            v = np.ascontiguousarray(values, dtype=np.float64).ravel()
            if v.size != self.qp_count():
                raise ValueError("material array must have one value per quadrature point")
            check(sgm_plan_set_material(self.h, which, v.ctypes.data, 0.0), "sgm_plan_set_material")

    def workspace_bytes(self):
        n = c_size_t()
        check(sgm_workspace_bytes(self.h, ctypes.byref(n)))
        return n.value

    def set_scheme(self, scheme):
        """1: mass-matrix Hodge stars (first scheme), 2: pairing solves (second scheme, default)."""
        check(sgm_plan_set_scheme(self.h, int(scheme)), "sgm_plan_set_scheme")

    def set_options(self, opts):
        """SGM_OPT_* bits (OPT_FULL_SCHEDULE, OPT_EXACT_SPIKE, OPT_SERIAL, OPT_NO_GRAPH, OPT_FUSED,
        OPT_WIDE_TILES, OPT_OTF_GEOMETRY)."""
        check(sgm_plan_set_options(self.h, int(opts)), "sgm_plan_set_options")

    def options(self):
        v = ctypes.c_uint(0)
        check(sgm_plan_get_options(self.h, ctypes.byref(v)), "sgm_plan_get_options")
        return v.value

    def schedule_mode(self):
        """0: full three-axis sweeps, 1: reduced separable schedule, 2: reduced with concurrent
        sweeps (default), 3: reduced with the update fused into the first sweeps (OPT_FUSED)."""
        v = c_int(0)
        check(sgm_plan_reduced_schedule(self.h, ctypes.byref(v)), "sgm_plan_reduced_schedule")
        return v.value

    def reduced_schedule(self):
        return self.schedule_mode() > 0

    def kernels_per_step(self):
        n = c_int()
        check(sgm_plan_kernels_per_step(self.h, ctypes.byref(n)))
        return n.value

    def set_profiling(self, on=True):
        check(sgm_plan_set_profiling(self.h, int(bool(on))), "sgm_plan_set_profiling")

    def profile(self):
        """{class name: (total ms, launches)} since the last call (event-timed on the stream)."""
        ms = (c_double * len(K_CLASSES))()
        cnt = (c_int * len(K_CLASSES))()
        check(sgm_plan_profile(self.h, ms, cnt), "sgm_plan_profile")
        return {K_CLASSES[i]: (ms[i], cnt[i]) for i in range(len(K_CLASSES)) if cnt[i]}

    def workspace(self):
        """The plan's device workspace (re-sized when set_material / set_scheme grow the need: the
        general Hodge's deterministic-accumulation scratch lives in it)."""
        nb = self.workspace_bytes()
        if self._ws is None or self._ws.numel() * 8 < nb:
            import torch
            self._ws = torch.empty((nb + 7) // 8, dtype=torch.float64, device=f"cuda:{self.device}")
        return self._ws

    # --- device calls (torch tensors or raw ints) ---
    def step(self, d, e, b, h, dt, n_steps=1, j_hat=None, j_amp=None, stream=None, ws=None):
        w = self.workspace() if ws is None else ws
        check(sgm_step(self.h, _ptr(d), _ptr(e), _ptr(b), _ptr(h), _ptr(j_hat), _ptr(j_amp), float(dt),
                       int(n_steps), _ptr(w), w.numel() * 8, _stream(stream)), "sgm_step")

    def step_lifted(self, d, e, b, h, dt, n_steps, g, beta, w_e=None, c_b=None, q0=None, q1=None, j_hat=None,
                    j_amp=None, stream=None, ws=None):
        """n_steps lifted steps (sgm_step_lifted): g, beta device arrays of n_steps; the precomputed
        lifting vectors w_e (N_e), c_b (N_b), q0, q1 (N_h) as device tensors or None."""
        w = self.workspace() if ws is None else ws
        L = sgm_lifting(_ptr(w_e), _ptr(c_b), _ptr(q0), _ptr(q1), _ptr(g), _ptr(beta))
        check(sgm_step_lifted(self.h, _ptr(d), _ptr(e), _ptr(b), _ptr(h), _ptr(j_hat), _ptr(j_amp), ctypes.byref(L),
                              float(dt), int(n_steps), _ptr(w), w.numel() * 8, _stream(stream)), "sgm_step_lifted")

    def step_eh(self, e, h, dt, n_steps=1, j_hat=None, j_amp=None, stream=None, ws=None):
        """The (e,h)-state variant (sgm_step_eh): only e and h are stored and advanced."""
        w = self.workspace() if ws is None else ws
        check(sgm_step_eh(self.h, _ptr(e), _ptr(h), _ptr(j_hat), _ptr(j_amp), float(dt), int(n_steps), _ptr(w),
                          w.numel() * 8, _stream(stream)), "sgm_step_eh")

    def step_composed(self, d, e, b, h, dt, weights=None, n_steps=1, j_hat=None, j_amp=None, stream=None,
                      ws=None):
        """Composition of kick-drift-kick sub-steps (sgm_step_composed); synchronous state.
        weights default: Yoshida's 4th-order triple jump (YOSHIDA4)."""
        w = self.workspace() if ws is None else ws
        wt = np.ascontiguousarray(YOSHIDA4 if weights is None else weights, dtype=np.float64)
        check(sgm_step_composed(self.h, _ptr(d), _ptr(e), _ptr(b), _ptr(h), _ptr(j_hat), _ptr(j_amp),
                                wt.ctypes.data, int(wt.size), float(dt), int(n_steps), _ptr(w), w.numel() * 8,
                                _stream(stream)), "sgm_step_composed")

    def step_host(self, d, e, b, h, dt, n_steps=1, j_hat=None, j_amp=None, stream=None):
        """d, e, b, h: numpy float64 arrays or pinned CPU torch tensors (updated in place)."""
        def hp(x):
            if x is None:
                return None
            if isinstance(x, np.ndarray):
                assert x.dtype == np.float64 and x.flags.c_contiguous
                return x.ctypes.data
            return x.data_ptr()
        check(sgm_step_host(self.h, hp(d), hp(e), hp(b), hp(h), hp(j_hat), hp(j_amp), float(dt), int(n_steps),
                            _stream(stream)), "sgm_step_host")

    def kron_solve(self, which, rhs, x, transpose=False, stream=None):
        w = self.workspace()
        check(sgm_kron_solve(self.h, which, int(transpose), _ptr(rhs), _ptr(x), _ptr(w), w.numel() * 8,
                             _stream(stream)), "sgm_kron_solve")

    def pairing_apply(self, which, x, y, transpose=False, stream=None):
        w = self.workspace()
        check(sgm_pairing_apply(self.h, which, int(transpose), _ptr(x), _ptr(y), _ptr(w), w.numel() * 8,
                                _stream(stream)), "sgm_pairing_apply")

    def hodge_apply(self, which, x, y, stream=None):
        w = self.workspace()
        check(sgm_hodge_apply(self.h, which, _ptr(x), _ptr(y), _ptr(w), w.numel() * 8, _stream(stream)),
              "sgm_hodge_apply")

    def hodge_star(self, which, x, y, stream=None):
        w = self.workspace()
        check(sgm_hodge_star(self.h, which, _ptr(x), _ptr(y), _ptr(w), w.numel() * 8, _stream(stream)),
              "sgm_hodge_star")

    def curl(self, kind, x, y, stream=None):
        check(sgm_curl(self.h, kind, _ptr(x), _ptr(y), _stream(stream)), "sgm_curl")

    def energy(self, d, e, b, h, out, stream=None):
        w = self.workspace()
        check(sgm_energy(self.h, _ptr(d), _ptr(e), _ptr(b), _ptr(h), _ptr(out), _ptr(w), w.numel() * 8,
                         _stream(stream)), "sgm_energy")

    def gauss(self, d, b, out, stream=None):
        w = self.workspace()
        check(sgm_gauss(self.h, _ptr(d), _ptr(b), _ptr(out), _ptr(w), w.numel() * 8, _stream(stream)),
              "sgm_gauss")

    def cfl(self, x, e, b, h, out, n_iter=300, stream=None):
        """Power-iteration leapfrog limit: out[0] = lambda, out[1] = dt_max (sgm_cfl)."""
        w = self.workspace()
        check(sgm_cfl(self.h, _ptr(x), _ptr(e), _ptr(b), _ptr(h), int(n_iter), _ptr(out), _ptr(w),
                      w.numel() * 8, _stream(stream)), "sgm_cfl")

    def check_source(self, j_hat, stream=None):
        w = self.workspace()
        return sgm_check_source(self.h, _ptr(j_hat), _ptr(w), w.numel() * 8, _stream(stream))
