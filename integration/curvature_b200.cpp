// curvature_b200.cpp -- the reference's curvature entry points on the B200 library.
//
// Drop-in replacement of /root/reference/proj/src/curvature.cpp: the same
// signatures (curvature.hpp:25-42), the same contract (memory cap,
// divisibility, exact symmetry, the pre-symmetrization asymmetry check), fp64
// arithmetic on the GPU through the C-ABI of include/curvkit_b200.h, errors
// mapped back onto the reference's classes (errors.hpp).  A curvkit build
// compiles this file instead of curvature.cpp and links -lcurvkit_b200.
//
// oracle/Makefile builds the reference's own acceptance suite
// (tests/acceptance.cpp) against it: tests/test_acceptance.py.
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "curv/curvature.hpp"
#include "curv/errors.hpp"
#include "curvkit_b200.h"

namespace curv {
namespace b200 {

// curv::ModelSpec (model.hpp:27-42) as the C-ABI's curvkit_model
struct Model {
    std::vector<int64_t> widths;
    curvkit_model m{};
    explicit Model(const ModelSpec& s) : widths(s.layer_widths.begin(), s.layer_widths.end()) {
        m.num_layers = (int32_t)widths.size();
        m.layer_widths = widths.data();
        m.hidden_activation = (int32_t)s.hidden_activation;  // Activation: identity, sigmoid, tanh, relu
        m.output_mode = (int32_t)s.output_mode;              // OutputMode: softmax_cross_entropy, raw_mean_output
    }
};

// curvkit_status -> the reference's exception classes
void check(int rc) {
    if (rc == CURVKIT_OK) return;
    const std::string msg = curvkit_last_error();
    switch (rc) {
        case CURVKIT_SHAPE_ERROR: throw ShapeError(msg);
        case CURVKIT_CONTRACT_ERROR: throw ContractError(msg);
        case CURVKIT_CONVERGENCE_ERROR: throw ConvergenceError(msg, {});
        default: throw std::runtime_error(msg);
    }
}

curvkit_curvature_config config(const CurvatureConfig& c) {
    return {(int64_t)c.batch_size_h, (int64_t)c.batch_size_g, (int64_t)c.parallelism, (int64_t)c.memory_cap};
}

// Batch rows n, with the reference's shape checks ahead of any device work
int64_t rows(const ModelSpec& spec, const Batch& b) {
    spec.validate();
    if (b.x.cols() != spec.input_width()) throw ShapeError("batch: input width does not match the model");
    if (b.y.rows() != b.x.rows() || b.y.cols() != spec.output_width())
        throw ShapeError("batch: target shape does not match the model");
    return (int64_t)b.size();
}

}  // namespace b200

HessianResult assemble_hessian(const ModelSpec& spec, const ParamVector& params, const Batch& dataset,
                               const CurvatureConfig& config) {
    b200::Model m(spec);
    const int64_t n = b200::rows(spec, dataset);
    const std::size_t p = param_count(spec);
    if (params.p() != p) throw ShapeError("assemble_hessian: parameter vector length does not match the model");
    HessianResult r{DenseMatrix(p, p), 0.0};
    const curvkit_curvature_config c = b200::config(config);
    // verify = 1: diagonal layer blocks from both triangles, the reference's
    // 1e-8 * max|H| asymmetry check (curvature.cpp:76-84), then symmetrized
    b200::check(curvkit_assemble_hessian(&m.m, params.data.data(), dataset.x.data(), dataset.y.data(), n, &c,
                                         CURVKIT_F64, /*verify=*/1, r.h.data(), &r.asymmetry));
    return r;
}

DenseMatrix assemble_jacobian(const ModelSpec& spec, const ParamVector& params, const Batch& batch) {
    if (batch.size() == 0) throw ContractError("assemble_jacobian: empty batch");
    b200::Model m(spec);
    const int64_t n = b200::rows(spec, batch);
    DenseMatrix j(batch.size(), param_count(spec));
    b200::check(curvkit_assemble_jacobian(&m.m, params.data.data(), batch.x.data(), batch.y.data(), n, CURVKIT_F64,
                                          j.data()));
    return j;
}

DenseMatrix assemble_opg(const ModelSpec& spec, const ParamVector& params, const Batch& dataset,
                         const CurvatureConfig& config) {
    b200::Model m(spec);
    const int64_t n = b200::rows(spec, dataset);
    const std::size_t p = param_count(spec);
    DenseMatrix g(p, p);
    const curvkit_curvature_config c = b200::config(config);
    b200::check(curvkit_assemble_opg(&m.m, params.data.data(), dataset.x.data(), dataset.y.data(), n, &c,
                                     CURVKIT_F64, g.data()));
    return g;
}

}  // namespace curv
