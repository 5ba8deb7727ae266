"""B200-native matrix-free SEM PCG (arXiv:1506.05996 / hexsem solver path).

The product is ``libhexsem_b200.so`` (C++ host setup + sm_100a CUDA kernels,
C-ABI in ``include/hexsem_b200.h``); this package is its Python host mirror.
"""
from .hexsem import (  # noqa: F401
    HexMesh,
    HeatConfig,
    build_heat_system,
    solve_heat,
    HostSetup,
    HxbError,
    Plan,
    ProblemConfig,
    build_system,
    derivation_matrix,
    fine_ops_model,
    fine_words_model,
    generate_box_mesh,
    generate_cube_mesh,
    gll,
    gll_nodes_weights,
    lib,
    make_mesh,
    mesh_info,
    mms_convergence,
    pencil,
    refine_uniform,
    residual_flops_model,
    residual_words_model,
    solve_poisson,
)
