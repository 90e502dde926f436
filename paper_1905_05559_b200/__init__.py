"""B200-native curvature library: exact Hessian, OPG and top-k OPG eigenpairs
of dense softmax-cross-entropy MLPs (arXiv 1905.05559), behind the reference
curvkit API.  Compute runs in libcurvkit_b200.so (sm_100a CUDA)."""
from .curv import (  # noqa: F401
    Activation, Batch, CurvatureConfig, EigenPairs, GradResult, HessianResult, HvpOperator, ModelSpec, OutputMode,
    assemble_hessian, assemble_jacobian, assemble_opg, bias_block_offset, default_lambda_tilde, eig_apply,
    flatten_params, full_rank_apply, full_rank_materialize, full_rank_quadform, grad_batch, hvp, low_rank_apply,
    low_rank_materialize, low_rank_quadform, opg_eigs, param_count, per_example_grad, unflatten_params,
    validate_eigen_pairs, weight_block_offset,
)
from .errors import ContractError, ConvergenceError, CurvError, ShapeError  # noqa: F401
