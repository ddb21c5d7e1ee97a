"""paper_2111_12238_b200 -- B200-native (sm_100a) executor for Sparse Fusion
(arXiv 2111.12238): fused execution of sparse kernel pairs with loop-carried
dependences, behind the reference's inspector/executor API.

The compute path is libsfgpu.so (CUDA, built in-tree by ``make -C
paper_2111_12238_b200``); this package is its Python face.  There is no CPU
fallback.
"""
from .api import (COMBOS, CscMatrix, DepDag, FactorizationError, FusedPartitioning,
                  FusedSchedule, InterDep, InvalidMatrixError, KernelState, LevelInfo,
                  NoDeviceError, PCG, ParseError, WavefrontSchedule, build_g1, build_g2,
                  build_wavefront_schedule, collect_outputs, compile_schedule,
                  compute_reuse, config5_systems, config_matrix, execute_fused,
                  execute_joint_wavefront, execute_sequential, execute_unfused,
                  gen_banded_spd, gen_grid_laplacian, gen_vector, inter_dag, joint_dag,
                  level_info, make_fused_schedule, make_state, msp, permute_symmetric,
                  read_matrix_market, read_permutation, reset, run_sequential_reference,
                  validate_fused_partitioning, write_matrix_market)

__all__ = [
    "COMBOS", "CscMatrix", "DepDag", "FactorizationError", "FusedPartitioning",
    "FusedSchedule", "InterDep", "InvalidMatrixError", "KernelState", "LevelInfo",
    "NoDeviceError", "PCG", "ParseError", "build_g1", "build_g2", "collect_outputs",
    "compute_reuse", "config5_systems", "config_matrix", "execute_fused",
    "execute_unfused", "gen_banded_spd", "gen_grid_laplacian", "gen_vector",
    "inter_dag", "joint_dag", "level_info", "make_fused_schedule",
    "make_state", "permute_symmetric", "read_matrix_market", "read_permutation",
    "reset", "write_matrix_market", "WavefrontSchedule", "build_wavefront_schedule",
    "compile_schedule", "execute_joint_wavefront", "execute_sequential", "msp",
    "run_sequential_reference", "validate_fused_partitioning",
]
