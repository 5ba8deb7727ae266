"""Python host mirror of the reference solver API over the B200 C-ABI.

Mirrors the reference's Python surface ``_hexsem`` (python/src/module.cpp:73-143:
``solve_poisson(**kwargs)``, ``mesh_info``, ``gll_nodes_weights``, counter
models) and its C++ objects (``HexMesh``, ``ProblemConfig``, ``SemSystem`` with
``operator_fn``/``preconditioner_fn``, ``pcg``) on top of
``libhexsem_b200.so`` (include/hexsem_b200.h). Every numeric operation runs
in the CUDA library; this module only marshals arguments. There is no CPU
fallback: if the library is missing or no sm_100 GPU is present, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HXB_LIB") or os.path.join(_HERE, "libhexsem_b200.so")  # HXB_LIB: A/B builds

FAMILIES = {"uniform": 0, "distorted_domain": 1, "distorted_elements": 2}
PRECONDS = {"two_scale": 0, "fine_only": 1, "coarse_only": 2, "none": 3}
COARSE = {"automatic": 0, "direct": 1, "amg": 2}
VARIANTS = {"stored": 0, "on_the_fly": 1}
TAGS = {"dirichlet": 0, "neumann": 1}
STATUS = {0: "converged", 1: "max_iterations", 2: "breakdown"}


class HxbError(RuntimeError):
    """Raised on a non-zero C-ABI return code (message from hxb_last_error)."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class _Mesh(C.Structure):
    _fields_ = [
        ("num_vertices", C.c_int32), ("xyz", C.POINTER(C.c_double)),
        ("num_elements", C.c_int32), ("conn", C.POINTER(C.c_int32)),
        ("num_boundary_faces", C.c_int32), ("bface_element", C.POINTER(C.c_int32)),
        ("bface_face", C.POINTER(C.c_int32)), ("bface_tag", C.POINTER(C.c_uint8)),
    ]


class _MeshBuf(C.Structure):
    _fields_ = [("view", _Mesh), ("impl", C.c_void_p)]


class _Options(C.Structure):
    _fields_ = [("precond_mode", C.c_int), ("coarse_solve", C.c_int), ("direct_threshold", C.c_int32),
                ("variant", C.c_int), ("device", C.c_int), ("bitwise_reference", C.c_int),
                ("n_gpus", C.c_int), ("devices", C.c_int * 8), ("rank", C.c_int), ("nranks", C.c_int),
                ("fused_combine", C.c_int), ("fdm_element_order", C.c_int), ("host_lists", C.c_int),
                ("restrict_in_fdm", C.c_int), ("coarse_sms", C.c_int), ("reserved", C.c_int * 2)]


class _PcgConfig(C.Structure):
    _fields_ = [("rel_tolerance", C.c_double), ("max_iterations", C.c_int), ("record_history", C.c_int)]


class _PcgResult(C.Structure):
    _fields_ = [("status", C.c_int), ("iterations", C.c_int), ("num_residuals", C.c_int), ("num_zr", C.c_int),
                ("residual_history", C.POINTER(C.c_double)), ("zr_history", C.POINTER(C.c_double)),
                ("u", C.POINTER(C.c_double)), ("solve_seconds", C.c_double), ("diagnostic", C.c_char * 256)]


class _HeatConfig(C.Structure):
    _fields_ = [("dt", C.c_double), ("steps", C.c_int), ("rho", C.c_double), ("cp", C.c_double),
                ("q_power", C.c_double), ("source_radius", C.c_double), ("has_source", C.c_int),
                ("auto_trajectory", C.c_int), ("source_start", C.c_double * 3), ("source_end", C.c_double * 3),
                ("initial_value", C.c_double)]


class _HeatStep(C.Structure):
    _fields_ = [("step", C.c_int), ("iterations", C.c_int), ("residual", C.c_double),
                ("mean_temperature", C.c_double), ("l2_norm", C.c_double), ("source_integral", C.c_double)]


class _PlanInfo(C.Structure):
    _fields_ = [("num_global", C.c_int64), ("num_elements", C.c_int64), ("num_vertices", C.c_int64),
                ("order", C.c_int32), ("coarse_uses_amg", C.c_int32), ("coarse_n", C.c_int64),
                ("amg_levels", C.c_int32), ("precond_mode", C.c_int32), ("amg_rows", C.c_int64 * 16),
                ("amg_nnz", C.c_int64 * 16), ("setup_seconds", C.c_double), ("device_bytes", C.c_int64),
                ("coarse_sms", C.c_int32), ("pad_", C.c_int32)]


# Exported symbols and their signatures (kept in sync with include/hexsem_b200.h).
P = C.c_void_p
SIGNATURES = {
    "hxb_last_error": (C.c_char_p, []),
    "hxb_default_options": (None, [C.POINTER(_Options)]),
    "hxb_generate_cube_mesh": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(C.POINTER(_MeshBuf))]),
    "hxb_generate_box_mesh": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double), C.c_int,
                                        C.POINTER(C.POINTER(_MeshBuf))]),
    "hxb_refine_uniform": (C.c_int, [C.POINTER(_Mesh), C.POINTER(C.POINTER(_MeshBuf))]),
    "hxb_mesh_free": (None, [C.POINTER(_MeshBuf)]),
    "hxb_read_mesh_file": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(C.POINTER(_MeshBuf))]),
    "hxb_write_mesh_file": (C.c_int, [C.POINTER(_Mesh), C.c_char_p, C.c_int]),
    "hxb_plan_create": (C.c_int, [C.POINTER(_Mesh), C.c_int, P, P, C.POINTER(_Options), C.POINTER(P)]),
    "hxb_plan_destroy": (C.c_int, [P]),
    "hxb_plan_get_info": (C.c_int, [P, C.POINTER(_PlanInfo)]),
    "hxb_apply_A": (C.c_int, [P, P, P]),
    "hxb_apply_P": (C.c_int, [P, P, P]),
    "hxb_apply_fine": (C.c_int, [P, P, P]),
    "hxb_apply_coarse": (C.c_int, [P, P, P]),
    "hxb_apply_A_device": (C.c_int, [P, C.c_void_p, C.c_void_p, C.c_void_p]),
    "hxb_apply_P_device": (C.c_int, [P, C.c_void_p, C.c_void_p, C.c_void_p]),
    "hxb_solve": (C.c_int, [P, P, C.POINTER(_PcgConfig), C.POINTER(_PcgResult)]),
    "hxb_solve_device": (C.c_int, [P, C.c_void_p, C.POINTER(_PcgConfig), C.POINTER(_PcgResult)]),
    "hxb_load_ones": (C.c_int, [P, P]),
    "hxb_solve_heat": (C.c_int, [P, C.POINTER(_HeatConfig), C.POINTER(_PcgConfig), C.POINTER(_HeatStep),
                                 C.POINTER(C.c_int), C.POINTER(C.c_int), P, C.POINTER(C.c_double)]),
    "hxb_node_coords": (C.c_int, [P, P]),
    "hxb_lumped_mass": (C.c_int, [P, P]),
    "hxb_export_geometry": (C.c_int, [P, P, P]),
    "hxb_export_maps": (C.c_int, [P, P, P, P, P, P, P]),
    "hxb_amg_level": (C.c_int, [P, C.c_int, P, P, P, P, P, P]),
    "hxb_bench_apply_A": (C.c_int, [P, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "hxb_profile": (C.c_int, [P, C.c_int, P]),
    "hxb_kernel_timing": (C.c_int, [P, C.c_int, C.c_int]),
    "hxb_kernel_timing_read": (C.c_int, [P, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int)]),
    "hxb_launch_count": (C.c_int, [P, C.POINTER(C.c_int64)]),
    "hxb_dist_info": (C.c_int, [P, P]),
    "hxb_dist_lists": (C.c_int, [P, P, P]),
    "hxb_dist_apply_A_begin": (C.c_int, [P, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "hxb_dist_apply_A_continue": (C.c_int, [P, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "hxb_dist_apply_A_end": (C.c_int, [P, C.c_void_p, C.c_void_p, C.c_void_p]),
    "hxb_dist_pcg_info": (C.c_int, [P, P]),
    "hxb_dist_vec": (C.c_int, [P, C.c_int, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "hxb_dist_dot": (C.c_int, [P, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "hxb_dist_pack": (C.c_int, [P, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "hxb_dist_unpack": (C.c_int, [P, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "hxb_dist_fine": (C.c_int, [P, C.c_void_p, C.c_void_p, C.c_void_p]),
    "hxb_dist_fine_recv": (C.c_int, [P, C.c_void_p, C.c_void_p]),
    "hxb_dist_rpart": (C.c_int, [P, C.c_int, C.c_void_p, C.c_void_p]),
    "hxb_dist_coarse": (C.c_int, [P, C.c_void_p]),
    "hxb_dist_combine": (C.c_int, [P, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "hxb_setup_create": (C.c_int, [C.POINTER(_Mesh), C.c_int, P, P, C.POINTER(_Options), C.POINTER(P)]),
    "hxb_setup_destroy": (None, [P]),
    "hxb_setup_info": (C.c_int, [P, C.POINTER(_PlanInfo)]),
    "hxb_setup_export_maps": (C.c_int, [P, P, P, P, P, P, P]),
    "hxb_setup_amg_level": (C.c_int, [P, C.c_int, P, P, P, P, P, P]),
    "hxb_setup_lumped_mass": (C.c_int, [P, P]),
    "hxb_setup_coarse_direct_check": (C.c_int, [P, P, P, P]),
    "hxb_setup_export_geometry": (C.c_int, [P, P, P]),
    "hxb_setup_dist_lists": (C.c_int, [P, C.c_int, C.c_int, P, P]),
    "hxb_gll": (C.c_int, [C.c_int, P, P, P]),
    "hxb_pencil": (C.c_int, [C.c_int, P, P, P, P, P]),
    "hxb_words_model": (C.c_uint64, [C.c_int64, C.c_int, C.c_int]),
    "hxb_flops_model": (C.c_uint64, [C.c_int64, C.c_int]),
    "hxb_fine_ops_model": (C.c_uint64, [C.c_int64, C.c_int]),
    "hxb_fine_words_model": (C.c_uint64, [C.c_int64, C.c_int]),
}

_lib = None


def lib():
    """Load libhexsem_b200.so (fails loudly: there is no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing; build it with `make -C paper_1506_05996_b200` "
                          "or __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def _check(rc: int):
    if rc != 0:
        raise HxbError(rc, lib().hxb_last_error().decode())


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------------------
@dataclass
class HexMesh:
    """Conforming all-hex mesh (mesh.hpp:38-45) as numpy arrays."""
    xyz: np.ndarray                      # (nv, 3) float64
    conn: np.ndarray                     # (ne, 8) int32, Gmsh corner order
    bf_elem: np.ndarray                  # (nbf,) int32
    bf_face: np.ndarray                  # (nbf,) int32
    bf_tag: np.ndarray                   # (nbf,) uint8 (0 dirichlet, 1 neumann)

    @property
    def num_elements(self) -> int:
        return int(self.conn.shape[0])

    @property
    def num_vertices(self) -> int:
        return int(self.xyz.shape[0])

    def as_dict(self) -> dict:
        return {"xyz": self.xyz, "conn": self.conn, "bf_elem": self.bf_elem, "bf_face": self.bf_face,
                "bf_tag": self.bf_tag}

    def _c(self) -> _Mesh:
        self.xyz = np.ascontiguousarray(self.xyz, dtype=np.float64)
        self.conn = np.ascontiguousarray(self.conn, dtype=np.int32)
        self.bf_elem = np.ascontiguousarray(self.bf_elem, dtype=np.int32)
        self.bf_face = np.ascontiguousarray(self.bf_face, dtype=np.int32)
        self.bf_tag = np.ascontiguousarray(self.bf_tag, dtype=np.uint8)
        m = _Mesh()
        m.num_vertices = self.num_vertices
        m.xyz = self.xyz.ctypes.data_as(C.POINTER(C.c_double))
        m.num_elements = self.num_elements
        m.conn = self.conn.ctypes.data_as(C.POINTER(C.c_int32))
        m.num_boundary_faces = int(self.bf_elem.size)
        m.bface_element = self.bf_elem.ctypes.data_as(C.POINTER(C.c_int32))
        m.bface_face = self.bf_face.ctypes.data_as(C.POINTER(C.c_int32))
        m.bface_tag = self.bf_tag.ctypes.data_as(C.POINTER(C.c_uint8))
        return m


def _take_mesh(buf) -> HexMesh:
    v = buf.contents.view
    nv, ne, nb = v.num_vertices, v.num_elements, v.num_boundary_faces
    m = HexMesh(
        xyz=np.ctypeslib.as_array(v.xyz, shape=(nv * 3,)).reshape(nv, 3).copy(),
        conn=np.ctypeslib.as_array(v.conn, shape=(ne * 8,)).reshape(ne, 8).copy(),
        bf_elem=np.ctypeslib.as_array(v.bface_element, shape=(max(nb, 1),))[:nb].copy(),
        bf_face=np.ctypeslib.as_array(v.bface_face, shape=(max(nb, 1),))[:nb].copy(),
        bf_tag=np.ctypeslib.as_array(v.bface_tag, shape=(max(nb, 1),))[:nb].copy(),
    )
    lib().hxb_mesh_free(buf)
    return m


def generate_cube_mesh(k: int, family: str = "uniform", boundary: str = "dirichlet") -> HexMesh:
    """generate_cube_mesh (mesh.hpp:53-54, mesh.cpp:110-139)."""
    out = C.POINTER(_MeshBuf)()
    _check(lib().hxb_generate_cube_mesh(k, FAMILIES[family], TAGS[boundary], C.byref(out)))
    return _take_mesh(out)


_MESHFILE = {"auto": 0, "msh": 1, "native": 2}


def read_mesh_file(path: str, fmt: str = "auto") -> HexMesh:
    """read_mesh_file / read_msh / read_native (mesh_io.cpp:49-124, 188-225)."""
    out = C.POINTER(_MeshBuf)()
    _check(lib().hxb_read_mesh_file(os.fsencode(path), _MESHFILE[fmt], C.byref(out)))
    return _take_mesh(out)


def write_mesh_file(mesh: HexMesh, path: str, fmt: str = "auto") -> None:
    """write_mesh_file / write_msh / write_native (mesh_io.cpp:126-186, 227-232)."""
    view = mesh._c()
    _check(lib().hxb_write_mesh_file(C.byref(view), os.fsencode(path), _MESHFILE[fmt]))


def read_msh(path: str) -> HexMesh:
    return read_mesh_file(path, "msh")


def write_msh(mesh: HexMesh, path: str) -> None:
    write_mesh_file(mesh, path, "msh")


def read_native(path: str) -> HexMesh:
    return read_mesh_file(path, "native")


def write_native(mesh: HexMesh, path: str) -> None:
    write_mesh_file(mesh, path, "native")


def generate_box_mesh(kx: int, ky: int, kz: int, size=(1.0, 1.0, 1.0), boundary: str = "dirichlet") -> HexMesh:
    """generate_box_mesh (mesh.hpp:57-58, mesh.cpp:67-108)."""
    out = C.POINTER(_MeshBuf)()
    sz = (C.c_double * 3)(*[float(x) for x in size])
    _check(lib().hxb_generate_box_mesh(kx, ky, kz, sz, TAGS[boundary], C.byref(out)))
    return _take_mesh(out)


def refine_uniform(mesh: HexMesh) -> HexMesh:
    """refine_uniform (mesh.hpp:60-62, mesh.cpp:141-234)."""
    out = C.POINTER(_MeshBuf)()
    cm = mesh._c()
    _check(lib().hxb_refine_uniform(C.byref(cm), C.byref(out)))
    return _take_mesh(out)


@dataclass
class ProblemConfig:
    """Solver-path subset of hexsem::ProblemConfig (problem.hpp:35-62)."""
    label: str = "poisson"
    mesh_file: str = ""
    family: str = "uniform"
    k: int = 8
    refine: int = 0
    bar: tuple = (0, 0, 0)
    bar_size: tuple = (1.0, 1.0, 8.0)
    boundary: str = "dirichlet"
    order: int = 3
    kappa: float = 1.0
    c: float = 0.0
    tol: float = 1e-6
    max_iterations: int = 500
    precond: str = "two_scale"
    variant: str = "stored"
    coarse_solve: str = "automatic"
    coarse_direct_threshold: int = 64000
    device: int = 0


def make_mesh(cfg: ProblemConfig) -> HexMesh:
    """make_mesh (problem.cpp:13-26): mesh file, box bar, or generated cube."""
    if cfg.mesh_file:
        mesh = read_mesh_file(cfg.mesh_file)
    elif cfg.bar[0] > 0:
        mesh = generate_box_mesh(cfg.bar[0], cfg.bar[1], cfg.bar[2], cfg.bar_size, cfg.boundary)
    else:
        mesh = generate_cube_mesh(cfg.k, cfg.family, cfg.boundary)
    for _ in range(cfg.refine):
        mesh = refine_uniform(mesh)
    return mesh


class Plan:
    """Device-resident SemSystem (problem.hpp:68-85): operator, two-scale
    preconditioner and PCG on one B200. Arrays in, arrays out."""

    def __init__(self, mesh: HexMesh, order: int, kappa_e=None, c_e=None, *, precond: str = "two_scale",
                 coarse_solve: str = "automatic", direct_threshold: int = 64000, variant: str = "stored",
                 device: int = 0, rank: int = 0, nranks: int = 1, split_combine: bool = True,
                 host_lists: bool = False, fdm_morton: bool = True, bitwise_reference: bool = False,
                 devices=None, restrict_in_fdm: bool = False, coarse_sms: int = 0):
        L = lib()
        ne = mesh.num_elements
        self.mesh = mesh
        self.kappa_e = np.ascontiguousarray(np.full(ne, 1.0) if kappa_e is None else kappa_e, dtype=np.float64)
        self.c_e = np.ascontiguousarray(np.zeros(ne) if c_e is None else c_e, dtype=np.float64)
        opt = _Options()
        L.hxb_default_options(C.byref(opt))
        opt.precond_mode = PRECONDS[precond]
        opt.coarse_solve = COARSE[coarse_solve]
        opt.direct_threshold = direct_threshold
        opt.variant = VARIANTS[variant]
        opt.device = device
        opt.rank = rank
        opt.nranks = nranks
        opt.fused_combine = 0 if split_combine else 1
        opt.host_lists = 1 if host_lists else 0
        opt.fdm_element_order = 0 if fdm_morton else 1
        opt.bitwise_reference = 1 if bitwise_reference else 0
        opt.restrict_in_fdm = 1 if restrict_in_fdm else 0
        opt.coarse_sms = int(coarse_sms)
        if devices is not None:  # multi-GPU plan: one element slab per entry (a device may repeat)
            if not 1 <= len(devices) <= 8:
                raise ValueError("devices: 1..8 entries")
            opt.n_gpus = len(devices)
            for r, d in enumerate(devices):
                opt.devices[r] = int(d)
            if len(devices) == 1:
                opt.device = int(devices[0])
        cm = mesh._c()
        h = C.c_void_p()
        _check(L.hxb_plan_create(C.byref(cm), order, _ptr(self.kappa_e), _ptr(self.c_e), C.byref(opt), C.byref(h)))
        self._h = h
        self.precond = precond
        info = _PlanInfo()
        _check(L.hxb_plan_get_info(self._h, C.byref(info)))
        self.N = int(info.num_global)
        self.NE = int(info.num_elements)
        self.NV = int(info.num_vertices)
        self.order = int(info.order)
        self.coarse_amg = bool(info.coarse_uses_amg)
        self.coarse_n = int(info.coarse_n)
        self.amg_levels = int(info.amg_levels)
        self.amg_rows = [int(info.amg_rows[i]) for i in range(self.amg_levels)]
        self.amg_nnz = [int(info.amg_nnz[i]) for i in range(self.amg_levels)]
        self.setup_seconds = float(info.setup_seconds)
        self.device_bytes = int(info.device_bytes)
        self.coarse_sms = int(info.coarse_sms)

    def close(self):
        if getattr(self, "_h", None):
            lib().hxb_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # --- LinearOp plug-ins (host arrays) ------------------------------------
    def _op(self, name, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.shape != (self.N,):
            raise ValueError(f"{name}: vector length mismatch")
        y = np.empty(self.N)
        _check(getattr(lib(), name)(self._h, _ptr(x), _ptr(y)))
        return y

    def apply_A(self, u):
        """SemOperator::apply (operator.cpp:255-287)."""
        return self._op("hxb_apply_A", u)

    def apply_P(self, r):
        """TwoScalePreconditioner::apply (precond.cpp:27-67)."""
        return self._op("hxb_apply_P", r)

    def apply_fine(self, r):
        """FinePreconditioner::apply on the masked residual (fine.cpp:210-231)."""
        return self._op("hxb_apply_fine", r)

    def apply_coarse(self, r):
        """CoarsePreconditioner::apply on the masked residual (coarse.cpp:188-208)."""
        return self._op("hxb_apply_coarse", r)

    def operator_fn(self):
        return self.apply_A

    def preconditioner_fn(self):
        return self.apply_P

    # --- device-pointer entry points (for the bench; data already in HBM) -----
    def apply_A_device(self, d_u: int, d_r: int, stream: int = 0):
        _check(lib().hxb_apply_A_device(self._h, C.c_void_p(d_u), C.c_void_p(d_r), C.c_void_p(stream or None)))

    def apply_P_device(self, d_r: int, d_z: int, stream: int = 0):
        _check(lib().hxb_apply_P_device(self._h, C.c_void_p(d_r), C.c_void_p(d_z), C.c_void_p(stream or None)))

    # --- solve ------------------------------------------------------------------
    def _solve(self, fn, bptr, tol, max_iterations, want_u=True, u_out=None):
        cfg = _PcgConfig(float(tol), int(max_iterations), 1)
        rh = np.zeros(max_iterations + 1)
        zh = np.zeros(max_iterations + 1)
        if u_out is not None:  # caller-owned (e.g. pinned) output buffer
            if u_out.dtype != np.float64 or u_out.shape != (self.N,) or not u_out.flags.c_contiguous:
                raise ValueError("pcg: u_out must be a contiguous float64 array of length N")
            want_u = True
        u = (u_out if u_out is not None else np.zeros(self.N)) if want_u else None
        res = _PcgResult()
        res.residual_history = rh.ctypes.data_as(C.POINTER(C.c_double))
        res.zr_history = zh.ctypes.data_as(C.POINTER(C.c_double))
        res.u = u.ctypes.data_as(C.POINTER(C.c_double)) if want_u else C.POINTER(C.c_double)()
        _check(fn(self._h, bptr, C.byref(cfg), C.byref(res)))
        return {"status": STATUS[res.status], "iterations": int(res.iterations),
                "residual_history": rh[:res.num_residuals].copy(), "zr_history": zh[:res.num_zr].copy(),
                "u": u, "solve_seconds": float(res.solve_seconds), "diagnostic": res.diagnostic.decode()}

    def pcg(self, b=None, tol: float = 1e-6, max_iterations: int = 500, want_u: bool = True, u_out=None) -> dict:
        """pcg(operator_fn, preconditioner_fn, b, cfg) (krylov.cpp:20-71) on the device.
        b=None uses the Poisson load m_N*1 masked (problem.cpp:129). u_out: optional
        caller-owned output array (pinned host memory makes the copies DMA-speed)."""
        bb = None if b is None else np.ascontiguousarray(b, dtype=np.float64)
        if bb is not None and bb.shape != (self.N,):
            raise ValueError("pcg: vector length mismatch")
        return self._solve(lib().hxb_solve, _ptr(bb), tol, max_iterations, want_u, u_out)

    def pcg_device(self, d_b: int | None, tol: float = 1e-6, max_iterations: int = 500, want_u: bool = False):
        return self._solve(lib().hxb_solve_device, C.c_void_p(d_b) if d_b else None, tol, max_iterations, want_u)

    def solve_heat(self, heat: "HeatConfig", tol: float = 1e-6, max_iterations: int = 500) -> dict:
        """solve_heat's time loop (problem.cpp:145-255) on this plan, which must
        carry c = 1/dt per element (build it with build_heat_system)."""
        hc = heat._c()
        cfg = _PcgConfig(float(tol), int(max_iterations), 1)
        steps = (_HeatStep * max(1, heat.steps))()
        ns, ok = C.c_int(), C.c_int()
        u = np.zeros(self.N)
        secs = C.c_double()
        _check(lib().hxb_solve_heat(self._h, C.byref(hc), C.byref(cfg), steps, C.byref(ns), C.byref(ok), _ptr(u),
                                    C.byref(secs)))
        rows = [{"step": st.step, "iterations": st.iterations, "residual": st.residual,
                 "mean_temperature": st.mean_temperature, "l2_norm": st.l2_norm,
                 "source_integral": st.source_integral} for st in steps[:ns.value]]
        return {"steps": rows, "all_converged": bool(ok.value), "final_field": u, "solve_seconds": secs.value}

    def node_coords(self):
        xyz = np.zeros(3 * self.N)
        _check(lib().hxb_node_coords(self._h, _ptr(xyz)))
        return xyz.reshape(self.N, 3)

    # --- data ---------------------------------------------------------------------
    def load_ones(self):
        b = np.empty(self.N)
        _check(lib().hxb_load_ones(self._h, _ptr(b)))
        return b

    def lumped_mass(self):
        m = np.empty(self.N)
        _check(lib().hxb_lumped_mass(self._h, _ptr(m)))
        return m

    def geometry(self, planes: bool = True) -> dict:
        """Device-computed factors of this plan's elements: mass (NE, nloc) and
        the six kappa*m*Gt planes (6, NE, nloc) (compute_factors, geometry.cpp:105-151)."""
        nloc = (self.order + 1) ** 3
        mass = np.empty(self.NE * nloc)
        wg = np.empty(6 * self.NE * nloc) if planes else None
        _check(lib().hxb_export_geometry(self._h, _ptr(mass), _ptr(wg)))
        return {"mass": mass.reshape(self.NE, nloc), "wg": None if wg is None else wg.reshape(6, self.NE, nloc)}

    def maps(self, sub: bool = True) -> dict:
        n = self.order
        nloc, nsub = (n + 1) ** 3, (n + 3) ** 3
        out = {
            "l2g": np.zeros(self.NE * nloc, dtype=np.int32),
            "g2l_offsets": np.zeros(self.N + 1, dtype=np.int64),
            "g2l_elem": np.zeros(self.NE * nloc, dtype=np.int32),
            "g2l_local": np.zeros(self.NE * nloc, dtype=np.int32),
            "sub_l2g": np.zeros(self.NE * nsub, dtype=np.int32) if sub else None,
            "dirichlet_mask": np.zeros(self.N, dtype=np.uint8),
        }
        _check(lib().hxb_export_maps(self._h, _ptr(out["l2g"]), _ptr(out["g2l_offsets"]), _ptr(out["g2l_elem"]),
                                     _ptr(out["g2l_local"]), _ptr(out["sub_l2g"]), _ptr(out["dirichlet_mask"])))
        return out

    def amg_level(self, l: int) -> dict:
        rows, nnz = C.c_int64(), C.c_int64()
        _check(lib().hxb_amg_level(self._h, l, C.byref(rows), C.byref(nnz), None, None, None, None))
        ptr = np.zeros(rows.value + 1, dtype=np.int64)
        col = np.zeros(nnz.value, dtype=np.int32)
        val = np.zeros(nnz.value)
        agg = np.full(rows.value, -1, dtype=np.int32)
        _check(lib().hxb_amg_level(self._h, l, C.byref(rows), C.byref(nnz), _ptr(ptr), _ptr(col), _ptr(val),
                                   _ptr(agg)))
        return {"ptr": ptr, "col": col, "val": val, "aggregate": agg}

    def profile(self, reps: int = 10) -> dict:
        """Per-component device times in ms (CUDA events, warm caches)."""
        out = np.zeros(16)
        _check(lib().hxb_profile(self._h, reps, _ptr(out)))
        keys = ["ax_elem", "ax_gather", "fdm", "coarse", "combine", "precond", "pcg_update", "pcg_dir",
                "restrict", "prolong", "amg", "amg_ksolve1_cluster", "combine_fine_only", "combine_coarse_only"]
        return dict(zip(keys, out.tolist()))

    # --- distributed operator (element-slab partition, hxb_dist_*) -------------
    def dist_info(self) -> dict:
        v = np.zeros(8, dtype=np.int64)
        _check(lib().hxb_dist_info(self._h, _ptr(v)))
        keys = ["rank", "nranks", "e0", "e1", "n_up", "n_down", "n_group0", "N"]
        return dict(zip(keys, (int(x) for x in v)))

    def dist_lists(self):
        info = self.dist_info()
        up = np.zeros(max(1, info["n_up"]), dtype=np.int32)
        down = np.zeros(max(1, info["n_down"]), dtype=np.int32)
        _check(lib().hxb_dist_lists(self._h, _ptr(up), _ptr(down)))
        return up[:info["n_up"]], down[:info["n_down"]]

    def dist_apply_A_begin(self, d_u: int, d_r: int, d_send_up: int, stream: int = 0):
        _check(lib().hxb_dist_apply_A_begin(self._h, C.c_void_p(d_u), C.c_void_p(d_r), C.c_void_p(d_send_up or None),
                                            C.c_void_p(stream or None)))

    def dist_apply_A_continue(self, d_u: int, d_r: int, d_recv_down: int, d_send_down: int, stream: int = 0):
        _check(lib().hxb_dist_apply_A_continue(self._h, C.c_void_p(d_u), C.c_void_p(d_r), C.c_void_p(d_recv_down or None),
                                               C.c_void_p(d_send_down or None), C.c_void_p(stream or None)))

    def dist_apply_A_end(self, d_r: int, d_recv_up: int, stream: int = 0):
        _check(lib().hxb_dist_apply_A_end(self._h, C.c_void_p(d_r), C.c_void_p(d_recv_up or None),
                                          C.c_void_p(stream or None)))

    def dist_pcg_info(self) -> dict:
        v = np.zeros(16, dtype=np.int64)
        _check(lib().hxb_dist_pcg_info(self._h, _ptr(v)))
        keys = ["ghost_from_down", "ghost_from_up", "ghost_to_down", "ghost_to_up", "fsend_down", "fsend_up",
                "frecv_down", "frecv_up", "e0", "e1", "ne_total", "has_fine", "has_coarse", "n_up", "n_down", "N"]
        return dict(zip(keys, (int(x) for x in v)))

    def dist_call(self, name: str, *args):
        """Raw staged call hxb_dist_<name>(plan, *args) (device pointers as ints)."""
        conv = [C.c_void_p(a) if isinstance(a, int) and not isinstance(a, bool) else a for a in args]
        _check(getattr(lib(), "hxb_dist_" + name)(self._h, *conv))

    KT_TAGS = {"ax_elem": 0, "ax_gather": 1, "fdm": 2, "combine": 3, "coarse": 4, "combine_fine": 5}

    def kernel_timing(self, enable: bool, max_launches: int = 4096):
        """Bracket tagged launches with CUDA events (hxb_kernel_timing)."""
        _check(lib().hxb_kernel_timing(self._h, 1 if enable else 0, int(max_launches)))

    def kernel_time(self, tag: str):
        """(total ms, launches) of one tagged kernel since kernel_timing(True)."""
        ms, cnt = C.c_double(), C.c_int()
        _check(lib().hxb_kernel_timing_read(self._h, self.KT_TAGS[tag], C.byref(ms), C.byref(cnt)))
        return ms.value, cnt.value

    def launch_count(self) -> int:
        n = C.c_int64()
        _check(lib().hxb_launch_count(self._h, C.byref(n)))
        return n.value

    def apply_A_host_ptr(self, h_u: int, h_r: int):
        """hxb_apply_A on raw (pinned) host pointers: H2D, Ax, D2H."""
        _check(lib().hxb_apply_A(self._h, C.c_void_p(h_u), C.c_void_p(h_r)))

    def bench_apply_A(self, reps: int = 20):
        ms, ms_elem = C.c_double(), C.c_double()
        _check(lib().hxb_bench_apply_A(self._h, reps, C.byref(ms), C.byref(ms_elem)))
        return ms.value, ms_elem.value


class HostSetup:
    """GPU-free setup (build_system minus the device upload): numbering,
    lumped mass, coarse matrix and AMG hierarchy, for bit-exact checks."""

    def __init__(self, mesh: HexMesh, order: int, kappa_e=None, c_e=None, *, precond: str = "two_scale",
                 coarse_solve: str = "automatic", direct_threshold: int = 64000):
        L = lib()
        ne = mesh.num_elements
        self.kappa_e = np.ascontiguousarray(np.full(ne, 1.0) if kappa_e is None else kappa_e, dtype=np.float64)
        self.c_e = np.ascontiguousarray(np.zeros(ne) if c_e is None else c_e, dtype=np.float64)
        opt = _Options()
        L.hxb_default_options(C.byref(opt))
        opt.precond_mode = PRECONDS[precond]
        opt.coarse_solve = COARSE[coarse_solve]
        opt.direct_threshold = direct_threshold
        cm = mesh._c()
        h = C.c_void_p()
        _check(L.hxb_setup_create(C.byref(cm), order, _ptr(self.kappa_e), _ptr(self.c_e), C.byref(opt), C.byref(h)))
        self._h = h
        info = _PlanInfo()
        _check(L.hxb_setup_info(self._h, C.byref(info)))
        self.N = int(info.num_global)
        self.NE = int(info.num_elements)
        self.NV = int(info.num_vertices)
        self.order = int(info.order)
        self.coarse_amg = bool(info.coarse_uses_amg)
        self.coarse_n = int(info.coarse_n)
        self.amg_levels = int(info.amg_levels)

    def close(self):
        if getattr(self, "_h", None):
            lib().hxb_setup_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def maps(self, sub: bool = True) -> dict:
        n = self.order
        nloc, nsub = (n + 1) ** 3, (n + 3) ** 3
        out = {
            "l2g": np.zeros(self.NE * nloc, dtype=np.int32),
            "g2l_offsets": np.zeros(self.N + 1, dtype=np.int64),
            "g2l_elem": np.zeros(self.NE * nloc, dtype=np.int32),
            "g2l_local": np.zeros(self.NE * nloc, dtype=np.int32),
            "sub_l2g": np.zeros(self.NE * nsub, dtype=np.int32) if sub else None,
            "dirichlet_mask": np.zeros(self.N, dtype=np.uint8),
        }
        _check(lib().hxb_setup_export_maps(self._h, _ptr(out["l2g"]), _ptr(out["g2l_offsets"]),
                                           _ptr(out["g2l_elem"]), _ptr(out["g2l_local"]), _ptr(out["sub_l2g"]),
                                           _ptr(out["dirichlet_mask"])))
        return out

    def amg_level(self, l: int) -> dict:
        rows, nnz = C.c_int64(), C.c_int64()
        _check(lib().hxb_setup_amg_level(self._h, l, C.byref(rows), C.byref(nnz), None, None, None, None))
        ptr = np.zeros(rows.value + 1, dtype=np.int64)
        col = np.zeros(nnz.value, dtype=np.int32)
        val = np.zeros(nnz.value)
        agg = np.full(rows.value, -1, dtype=np.int32)
        _check(lib().hxb_setup_amg_level(self._h, l, C.byref(rows), C.byref(nnz), _ptr(ptr), _ptr(col), _ptr(val),
                                         _ptr(agg)))
        return {"ptr": ptr, "col": col, "val": val, "aggregate": agg}

    def lumped_mass(self):
        m = np.empty(self.N)
        _check(lib().hxb_setup_lumped_mass(self._h, _ptr(m)))
        return m

    def coarse_direct_check(self) -> dict:
        """Sparse direct coarse factor (nested dissection + supernodal Cholesky,
        the device replacement of SimplicialLLT) checked on the host: relative
        residual of a solve with b = 1, stored factor entries, tree levels."""
        res, ent, lv = C.c_double(), C.c_int64(), C.c_int32()
        _check(lib().hxb_setup_coarse_direct_check(self._h, C.byref(res), C.byref(ent), C.byref(lv)))
        return {"rel_residual": res.value, "factor_entries": ent.value, "levels": lv.value}

    def geometry(self) -> dict:
        """Host restatement of compute_factors + kappa*mass scaling (setup_mesh.cpp)."""
        nloc = (self.order + 1) ** 3
        mass, wg = np.empty(self.NE * nloc), np.empty(6 * self.NE * nloc)
        _check(lib().hxb_setup_export_geometry(self._h, _ptr(mass), _ptr(wg)))
        return {"mass": mass.reshape(self.NE, nloc), "wg": wg.reshape(6, self.NE, nloc)}

    def dist_lists(self, rank: int, nranks: int) -> dict:
        """Element-slab partition lists of one rank (hxb_setup_dist_lists)."""
        cnt = np.zeros(6, dtype=np.int64)
        _check(lib().hxb_setup_dist_lists(self._h, rank, nranks, _ptr(cnt), None))
        nodes = np.zeros(max(1, int(cnt[5])), dtype=np.int32)
        _check(lib().hxb_setup_dist_lists(self._h, rank, nranks, _ptr(cnt), _ptr(nodes)))
        e0, e1, n0, nu, nd, nl = (int(x) for x in cnt)
        return {"e0": e0, "e1": e1, "group0": nodes[:n0], "up": nodes[n0:n0 + nu], "down": nodes[n0 + nu:nl]}


def gll(order: int):
    """GllBasis tables (gll.cpp:106-114): nodes, weights, D[i][j] = phi'_i(t_j)."""
    np1 = order + 1
    t, w, d = np.zeros(np1), np.zeros(np1), np.zeros(np1 * np1)
    _check(lib().hxb_gll(order, _ptr(t), _ptr(w), _ptr(d)))
    return t, w, d.reshape(np1, np1)


def gll_nodes_weights(n: int):
    t, w, _ = gll(n)
    return list(t), list(w)


def derivation_matrix(n: int):
    return gll(n)[2].tolist()


def pencil(order: int) -> dict:
    """PencilFactorization (fine.cpp:15-80)."""
    p = order + 3
    K, M, V, Vi, lam = np.zeros(p * p), np.zeros(p), np.zeros(p * p), np.zeros(p * p), np.zeros(p)
    _check(lib().hxb_pencil(order, _ptr(K), _ptr(M), _ptr(V), _ptr(Vi), _ptr(lam)))
    return {"K": K.reshape(p, p), "M": M, "V": V.reshape(p, p), "V_inv": Vi.reshape(p, p), "lambda": lam}


# ---------------------------------------------------------------------------
# Reference Python-module mirror (python/src/module.cpp)

def _config_from_kwargs(kw) -> ProblemConfig:
    cfg = ProblemConfig()
    for key in ("mesh_file", "k", "refine", "order", "kappa", "c", "family", "precond", "variant", "boundary", "tol",
                "max_iterations", "coarse_solve", "coarse_direct_threshold", "device", "label"):
        if key in kw:
            setattr(cfg, key, kw[key])
    if "bar" in kw:
        cfg.bar = tuple(kw["bar"])
    if "bar_size" in kw:
        cfg.bar_size = tuple(kw["bar_size"])
    return cfg


def build_system(config: ProblemConfig | None = None, **kw) -> Plan:
    """build_system (problem.cpp:73-108): kappa/c broadcast per element."""
    cfg = config or _config_from_kwargs(kw)
    mesh = make_mesh(cfg)
    ne = mesh.num_elements
    return Plan(mesh, cfg.order, np.full(ne, float(cfg.kappa)), np.full(ne, float(cfg.c)), precond=cfg.precond,
                coarse_solve=cfg.coarse_solve, direct_threshold=cfg.coarse_direct_threshold, variant=cfg.variant,
                device=cfg.device)


def solve_poisson(**kw) -> dict:
    """solve_poisson (problem.cpp:126-143 / module.cpp:106-114): s = 1."""
    cfg = _config_from_kwargs(kw)
    with build_system(cfg) as plan:
        res = plan.pcg(None, cfg.tol, cfg.max_iterations)
        report = {
            "label": cfg.label, "status": res["status"], "iterations": res["iterations"], "N": plan.N,
            "N_E": plan.NE, "n": plan.order, "residual_history": res["residual_history"].tolist(),
            "zr_history": res["zr_history"].tolist(),
            "operator": {"variant": cfg.variant, "n": plan.order, "N_E": plan.NE,
                         "flops_model": residual_flops_model(plan.NE, plan.order),
                         "bytes_model": residual_words_model(plan.NE, plan.order, cfg.variant) * 8},
            "timings": {"setup_seconds": plan.setup_seconds, "solve_seconds": res["solve_seconds"]},
        }
        if plan.coarse_n > 0:
            report["coarse"] = {"unknowns": plan.coarse_n, "solver": "amg" if plan.coarse_amg else "direct"}
            if plan.coarse_amg:
                report["coarse"]["hierarchy"] = {"levels": [{"rows": r, "nnz": z} for r, z in
                                                            zip(plan.amg_rows, plan.amg_nnz)]}
        if res["diagnostic"]:
            report["diagnostic"] = res["diagnostic"]
        return {"report": report, "u": res["u"]}


@dataclass
class HeatConfig:
    """HeatConfig (problem.hpp:18-31)."""
    dt: float = 0.04
    steps: int = 70
    rho: float = 7000.0
    cp: float = 0.8
    q_power: float = 1000.0
    source_radius: float = 0.5
    has_source: bool = True
    auto_trajectory: bool = True
    source_start: tuple = (0.0, 0.0, 0.0)
    source_end: tuple = (0.0, 0.0, 0.0)
    initial_value: float = 0.0

    def _c(self) -> _HeatConfig:
        h = _HeatConfig()
        h.dt, h.steps, h.rho, h.cp = float(self.dt), int(self.steps), float(self.rho), float(self.cp)
        h.q_power, h.source_radius = float(self.q_power), float(self.source_radius)
        h.has_source, h.auto_trajectory = int(bool(self.has_source)), int(bool(self.auto_trajectory))
        for d in range(3):
            h.source_start[d] = float(self.source_start[d])
            h.source_end[d] = float(self.source_end[d])
        h.initial_value = float(self.initial_value)
        return h


def build_heat_system(config: ProblemConfig, heat: HeatConfig) -> Plan:
    """build_system with c = 1/dt enforced (problem.cpp:148-150)."""
    if not heat.dt > 0:
        raise ValueError("heat: dt must be positive")
    mesh = make_mesh(config)
    ne = mesh.num_elements
    return Plan(mesh, config.order, np.full(ne, float(config.kappa)), np.full(ne, 1.0 / heat.dt),
                precond=config.precond, coarse_solve=config.coarse_solve,
                direct_threshold=config.coarse_direct_threshold, device=config.device)


def solve_heat(**kw) -> dict:
    """solve_heat (problem.cpp:145-255 / module.cpp:116-134) on the device."""
    cfg = _config_from_kwargs(kw)
    heat = HeatConfig()
    for key, name in (("dt", "dt"), ("steps", "steps"), ("rho", "rho"), ("cp", "cp"), ("Q", "q_power"),
                      ("q_power", "q_power"), ("source_radius", "source_radius"), ("has_source", "has_source"),
                      ("initial_value", "initial_value"), ("auto_trajectory", "auto_trajectory"),
                      ("source_start", "source_start"), ("source_end", "source_end")):
        if key in kw:
            setattr(heat, name, kw[key])
    with build_heat_system(cfg, heat) as plan:
        out = plan.solve_heat(heat, cfg.tol, cfg.max_iterations)
        out["N"] = plan.N
        return out


def mms_convergence(min_order: int = 1, max_order: int = 6, **kw) -> dict:
    """mms_convergence (problem.cpp:257-284 / module.cpp:129-133): u* = sin(pi x)
    sin(pi y) sin(pi z), s = 3 pi^2 kappa u*, all-Dirichlet, c = 0; per order
    the mass-weighted discrete L2 error of the device PCG solution."""
    cfg = _config_from_kwargs(kw)
    cfg.boundary = "dirichlet"
    cfg.c = 0.0
    rows = []
    for n in range(min_order, max_order + 1):
        cfg.order = n
        with build_system(cfg) as plan:
            x = plan.node_coords()
            ustar = np.sin(np.pi * x[:, 0]) * np.sin(np.pi * x[:, 1]) * np.sin(np.pi * x[:, 2])
            m = plan.lumped_mass()
            mask = plan.maps(sub=False)["dirichlet_mask"].astype(bool)
            s = 3 * np.pi * np.pi * cfg.kappa * ustar  # assemble_load (problem.cpp:38-46)
            b = np.where(mask, 0.0, m * s)
            res = plan.pcg(b, cfg.tol, cfg.max_iterations)
            d = res["u"] - ustar
            rows.append({"order": n, "num_global": plan.N, "error": float(np.sqrt(np.sum(m * d * d))),
                         "iterations": res["iterations"]})
    return {"rows": rows}


def write_mesh(path: str, **kw) -> None:
    """module.cpp:102-105: write_mesh_file(make_mesh(config), path)."""
    write_mesh_file(make_mesh(_config_from_kwargs(kw)), path)


def mesh_info(**kw) -> dict:
    cfg = _config_from_kwargs(kw)
    mesh = make_mesh(cfg)
    n = cfg.order
    hs = HostSetup(mesh, n, precond="none")  # build_index_maps only (module.cpp:91-101); no device needed
    try:
        return {"num_elements": mesh.num_elements, "num_vertices": mesh.num_vertices, "num_nodes": hs.N}
    finally:
        hs.close()


def residual_flops_model(ne: int, n: int) -> int:
    return int(lib().hxb_flops_model(ne, n))


def residual_words_model(ne: int, n: int, variant: str = "stored") -> int:
    return int(lib().hxb_words_model(ne, n, VARIANTS[variant]))


def fine_ops_model(ne: int, n: int) -> int:
    return int(lib().hxb_fine_ops_model(ne, n))


def fine_words_model(ne: int, n: int) -> int:
    return int(lib().hxb_fine_words_model(ne, n))


def synthetic_vector(n: int, seed: int = 12345) -> np.ndarray:
    """Synthetic input vector: splitmix64 values in [-0.5, 0.5), the generator
    the reference's tests feed its operators (random_vector,
    tests/support/oracles.cpp:126-139). Used by bench.py to build inputs."""
    M = np.uint64(0xFFFFFFFFFFFFFFFF)
    idx = np.arange(1, n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (np.uint64(seed) + idx * np.uint64(0x9E3779B97F4A7C15)) & M
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53) - 0.5
