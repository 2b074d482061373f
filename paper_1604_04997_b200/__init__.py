"""B200-native batched back end for kernelcost (arXiv 1604.04997).

The package is the hot path only: exact evaluation of a kernel's symbolic
operation counts over grids of parameter bindings, fused with the linear
run-time prediction, the argmin over kernel variants and the Gram reduction
of the least-squares fit. See DESIGN.md; the C ABI is include/kcg.h.
"""
from .api import (  # noqa: F401
    BoundBatch,
    Columns,
    EnumProgram,
    read_columns,
    write_columns,
    Grid,
    Prediction,
    predict_detail,
    grid_bindings,
    predict_grid,
    load_enum_program,
    KernelMeasurements,
    eval_from_csv,
    fit_from_csv,
    read_measurements,
    FitResult,
    GramStats,
    ModelWeights,
    Program,
    argmin,
    predict_host,
    predict_multi,
    multi_jit_source,
    evaluate_properties,
    fit_weights,
    geometric_mean_error,
    gram_accumulate,
    gram_fused,
    launch_count,
    measure_pipe_peak,
    measure_stream,
    load_program,
    noiseless_time,
    predict,
    read_weights_json,
    residual_fused,
    schema_index,
    schema_keys,
    schema_size,
    simulate_time,
    solve_gram,
    suite_index,
    write_weights_json,
)
from ._capi import KcgError  # noqa: F401
