"""ctypes bindings for the two CPU checkers (TEST INFRASTRUCTURE ONLY).

``libhexsem_ref.so`` (prefix ``ref_``) is the compiled reference;
``libhexsem_oracle.so`` (prefix ``orc_``) is the restatement. Both export the
same C-ABI (see oracle/ref_driver.cpp), so one wrapper class serves both.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_REF_SO = os.path.join(_HERE, "_ref", "libhexsem_ref.so")
_ORC_SO = os.path.join(_HERE, "_ref", "libhexsem_oracle.so")
_ORC_FMA_SO = os.path.join(_HERE, "_ref", "libhexsem_oracle_fma.so")

FAMILIES = {"uniform": 0, "distorted_domain": 1, "distorted_elements": 2}
PRECONDS = {"two_scale": 0, "fine_only": 1, "coarse_only": 2, "none": 3}
VARIANTS = {"stored": 0, "on_the_fly": 1}
COARSE = {"automatic": 0, "direct": 1, "amg": 2}
BOUNDARY = {"dirichlet": 0, "neumann": 1}
STATUS = {0: "converged", 1: "max_iterations", 2: "breakdown"}


class _CConfig(C.Structure):
    _fields_ = [
        ("k", C.c_int), ("refine", C.c_int), ("family", C.c_int), ("boundary", C.c_int),
        ("bar", C.c_int * 3), ("bar_size", C.c_double * 3),
        ("order", C.c_int), ("kappa", C.c_double), ("c", C.c_double),
        ("precond", C.c_int), ("variant", C.c_int), ("coarse_solve", C.c_int),
        ("coarse_direct_threshold", C.c_int),
        ("concurrent_precond", C.c_int), ("fine_threads", C.c_int),
    ]


@dataclass
class RefConfig:
    """Mirror of hexsem::ProblemConfig (problem.hpp:35-62)."""
    k: int = 8
    refine: int = 0
    family: str = "uniform"
    boundary: str = "dirichlet"
    bar: tuple = (0, 0, 0)
    bar_size: tuple = (1.0, 1.0, 8.0)
    order: int = 3
    kappa: float = 1.0
    c: float = 0.0
    precond: str = "two_scale"
    variant: str = "stored"
    coarse_solve: str = "automatic"
    coarse_direct_threshold: int = 64000
    concurrent_precond: bool = False
    fine_threads: int = 1

    def to_c(self) -> _CConfig:
        c = _CConfig()
        c.k, c.refine = self.k, self.refine
        c.family, c.boundary = FAMILIES[self.family], BOUNDARY[self.boundary]
        for d in range(3):
            c.bar[d] = int(self.bar[d])
            c.bar_size[d] = float(self.bar_size[d])
        c.order, c.kappa, c.c = self.order, float(self.kappa), float(self.c)
        c.precond, c.variant = PRECONDS[self.precond], VARIANTS[self.variant]
        c.coarse_solve = COARSE[self.coarse_solve]
        c.coarse_direct_threshold = self.coarse_direct_threshold
        c.concurrent_precond = int(self.concurrent_precond)
        c.fine_threads = self.fine_threads
        return c


_libs: dict = {}


def _load(path: str, prefix: str):
    key = (path, prefix)
    if key in _libs:
        return _libs[key]
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
    lib = C.CDLL(path)
    P = C.c_void_p
    dp = C.POINTER(C.c_double)
    for name, res, args in [
        ("last_error", C.c_char_p, []),
        ("create", C.c_int, [C.POINTER(_CConfig), C.POINTER(P)]),
        ("create_mesh", C.c_int, [C.c_int, dp, C.c_int, P, C.c_int, P, P, P, C.c_int, dp, dp,
                                  C.POINTER(_CConfig), C.POINTER(P)]),
        ("destroy", None, [P]),
        ("info", C.c_int, [P, P]),
        ("export_mesh", C.c_int, [P, P, P, P, P, P]),
        ("export_maps", C.c_int, [P, P, P, P, P, P, P]),
        ("apply_A", C.c_int, [P, P, P]),
        ("apply_P", C.c_int, [P, P, P]),
        ("apply_fine", C.c_int, [P, P, P]),
        ("apply_coarse", C.c_int, [P, P, P]),
        ("restrict", C.c_int, [P, P, P]),
        ("prolongate", C.c_int, [P, P, P]),
        ("lumped_mass", C.c_int, [P, P]),
        ("load_ones", C.c_int, [P, P]),
        ("coarse_matrix", C.c_int, [P, P, P, P, P]),
        ("amg_level", C.c_int, [P, C.c_int, P, P, P, P, P, P]),
        ("pcg", C.c_int, [P, P, C.c_double, C.c_int, P, P, P, P, P, P]),
        ("gll", C.c_int, [C.c_int, P, P, P, P]),
        ("pencil", C.c_int, [C.c_int, P, P, P, P, P]),
        ("element_h", C.c_int, [P, P]),
        ("words_model", C.c_ulonglong, [C.c_longlong, C.c_int, C.c_int]),
        ("flops_model", C.c_ulonglong, [C.c_longlong, C.c_int]),
        ("fine_ops_model", C.c_ulonglong, [C.c_longlong, C.c_int]),
        ("fine_words_model", C.c_ulonglong, [C.c_longlong, C.c_int]),
    ]:
        fn = getattr(lib, prefix + name)
        fn.restype = res
        fn.argtypes = args
    _libs[key] = lib
    return lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


class _System:
    PATH = ""
    PREFIX = ""

    def __init__(self, config: RefConfig | None = None, *, mesh=None, order=None,
                 kappa_e=None, c_e=None, **kw):
        self.lib = _load(self.PATH, self.PREFIX)
        cfg = config or RefConfig(**kw)
        self.config = cfg
        h = C.c_void_p()
        cc = cfg.to_c()
        if mesh is None:
            rc = self._fn("create")(C.byref(cc), C.byref(h))
        else:
            xyz = np.ascontiguousarray(mesh["xyz"], dtype=np.float64).reshape(-1)
            conn = np.ascontiguousarray(mesh["conn"], dtype=np.int32).reshape(-1)
            be = np.ascontiguousarray(mesh["bf_elem"], dtype=np.int32)
            bf = np.ascontiguousarray(mesh["bf_face"], dtype=np.int32)
            bt = np.ascontiguousarray(mesh["bf_tag"], dtype=np.uint8)
            ne = conn.size // 8
            ka = np.ascontiguousarray(kappa_e if kappa_e is not None else np.full(ne, cfg.kappa), dtype=np.float64)
            ca = np.ascontiguousarray(c_e if c_e is not None else np.full(ne, cfg.c), dtype=np.float64)
            self._keep = (xyz, conn, be, bf, bt, ka, ca)
            rc = self._fn("create_mesh")(
                xyz.size // 3, xyz.ctypes.data_as(C.POINTER(C.c_double)), ne, _ptr(conn), be.size,
                _ptr(be), _ptr(bf), _ptr(bt), order if order is not None else cfg.order,
                ka.ctypes.data_as(C.POINTER(C.c_double)), ca.ctypes.data_as(C.POINTER(C.c_double)),
                C.byref(cc), C.byref(h))
        self._check(rc)
        self.h = h
        info = np.zeros(10, dtype=np.int64)
        self._check(self._fn("info")(self.h, _ptr(info)))
        (self.N, self.NE, self.NV, self.order, self.coarse_n, self.coarse_amg, self.amg_levels,
         self.nbf, build_ms, self.has_fine) = [int(x) for x in info]
        self.build_seconds = build_ms / 1000.0

    def _fn(self, name):
        return getattr(self.lib, self.PREFIX + name)

    def _check(self, rc):
        if rc != 0:
            msg = self._fn("last_error")().decode()
            raise (ValueError if rc == 1 else RuntimeError)(msg)

    def close(self):
        if getattr(self, "h", None):
            self._fn("destroy")(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --- exports ---------------------------------------------------------
    def mesh(self) -> dict:
        xyz = np.zeros((self.NV, 3))
        conn = np.zeros((self.NE, 8), dtype=np.int32)
        be = np.zeros(self.nbf, dtype=np.int32)
        bf = np.zeros(self.nbf, dtype=np.int32)
        bt = np.zeros(self.nbf, dtype=np.uint8)
        self._check(self._fn("export_mesh")(self.h, _ptr(xyz), _ptr(conn), _ptr(be), _ptr(bf), _ptr(bt)))
        return {"xyz": xyz, "conn": conn, "bf_elem": be, "bf_face": bf, "bf_tag": bt}

    def maps(self, sub=True) -> dict:
        n = self.order
        nloc = (n + 1) ** 3
        nsub = (n + 3) ** 3
        out = {
            "l2g": np.zeros(self.NE * nloc, dtype=np.int32),
            "g2l_offsets": np.zeros(self.N + 1, dtype=np.int64),
            "g2l_elem": np.zeros(self.NE * nloc, dtype=np.int32),
            "g2l_local": np.zeros(self.NE * nloc, dtype=np.int32),
            "sub_l2g": np.zeros(self.NE * nsub, dtype=np.int32) if sub else None,
            "dirichlet_mask": np.zeros(self.N, dtype=np.uint8),
        }
        self._check(self._fn("export_maps")(
            self.h, _ptr(out["l2g"]), _ptr(out["g2l_offsets"]), _ptr(out["g2l_elem"]),
            _ptr(out["g2l_local"]), _ptr(out["sub_l2g"]), _ptr(out["dirichlet_mask"])))
        return out

    def _vec_op(self, name, x, nout=None):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(nout if nout is not None else self.N)
        self._check(self._fn(name)(self.h, _ptr(x), _ptr(y)))
        return y

    def apply_A(self, u):
        return self._vec_op("apply_A", u)

    def apply_P(self, r):
        return self._vec_op("apply_P", r)

    def apply_fine(self, r):
        return self._vec_op("apply_fine", r)

    def apply_coarse(self, r):
        return self._vec_op("apply_coarse", r)

    def restrict(self, r):
        return self._vec_op("restrict", r, self.NV)

    def prolongate(self, Z):
        return self._vec_op("prolongate", Z, self.N)

    def lumped_mass(self):
        y = np.zeros(self.N)
        self._check(self._fn("lumped_mass")(self.h, _ptr(y)))
        return y

    def load_ones(self):
        y = np.zeros(self.N)
        self._check(self._fn("load_ones")(self.h, _ptr(y)))
        return y

    def element_h(self):
        y = np.zeros((self.NE, 3))
        self._check(self._fn("element_h")(self.h, _ptr(y)))
        return y

    def coarse_matrix(self):
        nnz = C.c_int64()
        self._check(self._fn("coarse_matrix")(self.h, C.byref(nnz), None, None, None))
        ptr = np.zeros(self.NV + 1, dtype=np.int64)
        col = np.zeros(nnz.value, dtype=np.int32)
        val = np.zeros(nnz.value)
        self._check(self._fn("coarse_matrix")(self.h, C.byref(nnz), _ptr(ptr), _ptr(col), _ptr(val)))
        return ptr, col, val

    def amg_level(self, l):
        rows, nnz = C.c_int64(), C.c_int64()
        self._check(self._fn("amg_level")(self.h, l, C.byref(rows), C.byref(nnz), None, None, None, None))
        ptr = np.zeros(rows.value + 1, dtype=np.int64)
        col = np.zeros(nnz.value, dtype=np.int32)
        val = np.zeros(nnz.value)
        agg = np.full(rows.value, -1, dtype=np.int32)
        self._check(self._fn("amg_level")(self.h, l, C.byref(rows), C.byref(nnz), _ptr(ptr),
                                          _ptr(col), _ptr(val), _ptr(agg)))
        return {"ptr": ptr, "col": col, "val": val, "aggregate": agg}

    def pcg(self, b, tol=1e-6, max_iterations=500) -> dict:
        b = np.ascontiguousarray(b, dtype=np.float64)
        it, st = C.c_int(), C.c_int()
        rh = np.zeros(max_iterations + 1)
        zh = np.zeros(max_iterations + 1)
        u = np.zeros(self.N)
        secs = C.c_double()
        self._check(self._fn("pcg")(self.h, _ptr(b), tol, max_iterations, C.byref(it), C.byref(st),
                                    _ptr(rh), _ptr(zh), _ptr(u), C.byref(secs)))
        k = it.value
        nres = k + 1 if np.linalg.norm(b) > 0 else 1
        return {"iterations": k, "status": STATUS[st.value], "residual_history": rh[:nres],
                "zr_history": zh[:k if st.value != 2 else k + 1], "u": u,
                "solve_seconds": secs.value}


class RefSystem(_System):
    """The compiled reference (oracle/_ref/libhexsem_ref.so)."""
    PATH = _REF_SO
    PREFIX = "ref_"


class OracleSystem(_System):
    """The plain C++ restatement (oracle/_ref/libhexsem_oracle.so)."""
    PATH = _ORC_SO
    PREFIX = "orc_"


class OracleFmaSystem(_System):
    """The restatement compiled with FMA contraction: a rounding-only
    perturbation of the reference, used to calibrate parity tolerances."""
    PATH = _ORC_FMA_SO
    PREFIX = "orc_"


def oracle_fma_available() -> bool:
    return os.path.exists(_ORC_FMA_SO)


class _CHeat(C.Structure):
    _fields_ = [("dt", C.c_double), ("steps", C.c_int), ("rho", C.c_double), ("cp", C.c_double),
                ("q_power", C.c_double), ("source_radius", C.c_double), ("has_source", C.c_int),
                ("auto_trajectory", C.c_int), ("source_start", C.c_double * 3), ("source_end", C.c_double * 3),
                ("initial_value", C.c_double)]


def ref_solve_heat(config: RefConfig, heat: dict, tol: float = 1e-6, max_iterations: int = 500) -> dict:
    """The reference's own solve_heat (problem.cpp:145-255) via oracle/_ref."""
    L = C.CDLL(_REF_SO)
    fn = L.ref_solve_heat
    fn.restype = C.c_int
    n = RefSystem(config).N
    h = _CHeat()
    h.dt, h.steps = float(heat.get("dt", 0.04)), int(heat.get("steps", 70))
    h.rho, h.cp = float(heat.get("rho", 7000.0)), float(heat.get("cp", 0.8))
    h.q_power, h.source_radius = float(heat.get("q_power", 1000.0)), float(heat.get("source_radius", 0.5))
    h.has_source, h.auto_trajectory = int(heat.get("has_source", True)), int(heat.get("auto_trajectory", True))
    for d in range(3):
        h.source_start[d] = float(heat.get("source_start", (0, 0, 0))[d])
        h.source_end[d] = float(heat.get("source_end", (0, 0, 0))[d])
    h.initial_value = float(heat.get("initial_value", 0.0))
    S = max(1, h.steps)
    its = np.zeros(S, dtype=np.int32)
    res, mean, l2, src = (np.zeros(S) for _ in range(4))
    u = np.zeros(n)
    ns, ok = C.c_int(), C.c_int()
    nout = C.c_int64()
    secs = C.c_double()
    cc = config.to_c()
    rc = fn(C.byref(cc), C.byref(h), C.c_double(tol), C.c_int(max_iterations), C.c_int64(n), C.byref(ns), C.byref(ok),
            _ptr(its), _ptr(res), _ptr(mean), _ptr(l2), _ptr(src), _ptr(u), C.byref(nout), C.byref(secs))
    if rc:
        L.ref_last_error.restype = C.c_char_p
        raise RuntimeError(L.ref_last_error().decode())
    k = ns.value
    rows = [{"step": q + 1, "iterations": int(its[q]), "residual": float(res[q]), "mean_temperature": float(mean[q]),
             "l2_norm": float(l2[q]), "source_integral": float(src[q])} for q in range(k)]
    return {"steps": rows, "all_converged": bool(ok.value), "final_field": u, "solve_seconds": secs.value}


_MESHFMT = {"auto": 0, "msh": 1, "native": 2}


def _ref_mesh_lib():
    lib = _load(RefSystem.PATH, RefSystem.PREFIX)
    if not getattr(lib, "_mesh_bound", False):
        P = C.c_void_p
        lib.ref_write_mesh.restype = C.c_int
        lib.ref_write_mesh.argtypes = [C.c_int, P, C.c_int, P, C.c_int, P, P, P, C.c_char_p, C.c_int]
        lib.ref_read_mesh.restype = C.c_int
        lib.ref_read_mesh.argtypes = [C.c_char_p, C.c_int, C.POINTER(P)]
        lib.ref_mesh_counts.argtypes = [P, P]
        lib.ref_mesh_export.argtypes = [P, P, P, P, P, P]
        lib.ref_mesh_free.argtypes = [P]
        lib._mesh_bound = True
    return lib


def ref_write_mesh(mesh: dict, path: str, fmt: str = "auto") -> None:
    """The reference's write_mesh_file / write_msh / write_native (mesh_io.cpp)."""
    lib = _ref_mesh_lib()
    xyz = np.ascontiguousarray(mesh["xyz"], dtype=np.float64)
    conn = np.ascontiguousarray(mesh["conn"], dtype=np.int32)
    be = np.ascontiguousarray(mesh["bf_elem"], dtype=np.int32)
    bf = np.ascontiguousarray(mesh["bf_face"], dtype=np.int32)
    bt = np.ascontiguousarray(mesh["bf_tag"], dtype=np.uint8)
    rc = lib.ref_write_mesh(xyz.shape[0], _ptr(xyz), conn.shape[0], _ptr(conn), be.size, _ptr(be), _ptr(bf),
                            _ptr(bt), os.fsencode(path), _MESHFMT[fmt])
    if rc:
        raise RuntimeError(lib.ref_last_error().decode())


def ref_read_mesh(path: str, fmt: str = "auto") -> dict:
    """The reference's read_mesh_file / read_msh / read_native (mesh_io.cpp)."""
    lib = _ref_mesh_lib()
    h = C.c_void_p()
    if lib.ref_read_mesh(os.fsencode(path), _MESHFMT[fmt], C.byref(h)):
        raise RuntimeError(lib.ref_last_error().decode())
    try:
        c = np.zeros(3, dtype=np.int64)
        lib.ref_mesh_counts(h, _ptr(c))
        nv, ne, nb = (int(x) for x in c)
        out = {"xyz": np.zeros((nv, 3)), "conn": np.zeros((ne, 8), dtype=np.int32),
               "bf_elem": np.zeros(nb, dtype=np.int32), "bf_face": np.zeros(nb, dtype=np.int32),
               "bf_tag": np.zeros(nb, dtype=np.uint8)}
        lib.ref_mesh_export(h, *(_ptr(out[k]) for k in ("xyz", "conn", "bf_elem", "bf_face", "bf_tag")))
        return out
    finally:
        lib.ref_mesh_free(h)


def ref_available() -> bool:
    return os.path.exists(_REF_SO)


def oracle_available() -> bool:
    return os.path.exists(_ORC_SO)


def _gll(path, prefix, n):
    lib = _load(path, prefix)
    np1 = n + 1
    nodes, weights = np.zeros(np1), np.zeros(np1)
    D, B = np.zeros(np1 * np1), np.zeros(8 * np1 ** 3)
    rc = getattr(lib, prefix + "gll")(n, _ptr(nodes), _ptr(weights), _ptr(D), _ptr(B))
    if rc:
        raise ValueError(getattr(lib, prefix + "last_error")().decode())
    return nodes, weights, D.reshape(np1, np1), B.reshape(8, np1 ** 3)


def _pencil(path, prefix, n):
    lib = _load(path, prefix)
    p = n + 3
    K, M, V, Vi, lam = np.zeros(p * p), np.zeros(p), np.zeros(p * p), np.zeros(p * p), np.zeros(p)
    rc = getattr(lib, prefix + "pencil")(n, _ptr(K), _ptr(M), _ptr(V), _ptr(Vi), _ptr(lam))
    if rc:
        raise ValueError(getattr(lib, prefix + "last_error")().decode())
    return {"K": K.reshape(p, p), "M": M, "V": V.reshape(p, p), "V_inv": Vi.reshape(p, p), "lambda": lam}


def ref_gll(n):
    return _gll(_REF_SO, "ref_", n)


def oracle_gll(n):
    return _gll(_ORC_SO, "orc_", n)


def ref_pencil(n):
    return _pencil(_REF_SO, "ref_", n)


def oracle_pencil(n):
    return _pencil(_ORC_SO, "orc_", n)


def _model(name, *a):
    path, prefix = (_REF_SO, "ref_") if ref_available() else (_ORC_SO, "orc_")
    return int(getattr(_load(path, prefix), prefix + name)(*a))


def words_model(ne, n, variant="stored"):
    return _model("words_model", ne, n, VARIANTS[variant])


def flops_model(ne, n):
    return _model("flops_model", ne, n)


def fine_ops_model(ne, n):
    return _model("fine_ops_model", ne, n)


def fine_words_model(ne, n):
    return _model("fine_words_model", ne, n)


def splitmix_vector(n: int, seed: int = 12345) -> np.ndarray:
    """random_vector of tests/support/oracles.cpp:126-139 (splitmix64, [-0.5, 0.5))."""
    M = np.uint64(0xFFFFFFFFFFFFFFFF)
    idx = np.arange(1, n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (np.uint64(seed) + idx * np.uint64(0x9E3779B97F4A7C15)) & M
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53) - 0.5
