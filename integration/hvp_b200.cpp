// hvp_b200.cpp -- curv::hvp (autodiff.hpp:60-65) on the B200 library.
//
// autodiff.cpp defines hvp next to the forward/backward code the rest of the
// reference still uses, so a maintainer would replace that one function body
// with the call below.  To run the reference's own acceptance suite against
// it WITHOUT editing the reference sources, oracle/Makefile links with
// -Wl,--wrap on hvp's mangled name: the suite's calls land here, autodiff.cpp
// stays as it is.
#include <cstdint>
#include <vector>

#include "curv/autodiff.hpp"
#include "curv/errors.hpp"
#include "curvkit_b200.h"

namespace curv {
namespace b200 {
void check(int rc);
}

// H_batch v of the batch-averaged cost, fp64 on the GPU (batched R-op)
DenseVector hvp_b200(const ModelSpec& spec, const ParamVector& params, const Batch& batch, const DenseVector& v) {
    spec.validate();
    const std::vector<int64_t> w(spec.layer_widths.begin(), spec.layer_widths.end());
    const curvkit_model m{(int32_t)w.size(), w.data(), (int32_t)spec.hidden_activation, (int32_t)spec.output_mode};
    if (v.len() != param_count(spec)) throw ShapeError("hvp: direction length does not match the model");
    if (batch.x.cols() != spec.input_width()) throw ShapeError("hvp: input width does not match the model");
    DenseVector out(v.len());
    b200::check(curvkit_hvp(&m, params.data.data(), batch.x.data(), batch.y.data(), (int64_t)batch.size(), v.data(), 1,
                            CURVKIT_F64, out.data()));
    return out;
}

}  // namespace curv

// the --wrap target for curv::hvp(ModelSpec const&, ParamVector const&, Batch const&, DenseVector const&)
extern "C" curv::DenseVector __wrap__ZN4curv3hvpERKNS_9ModelSpecERKNS_11ParamVectorERKNS_5BatchERKNS_11DenseVectorE(
    const curv::ModelSpec& spec, const curv::ParamVector& params, const curv::Batch& batch, const curv::DenseVector& v) {
    return curv::hvp_b200(spec, params, batch, v);
}
