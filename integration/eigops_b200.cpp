// eigops_b200.cpp -- the consumers of eigenpairs (eigensolve.hpp:19-20, 83-97:
// validate_eigen_pairs, low_rank_* and full_rank_*) on the B200 library.
//
// eigensolve.cpp defines them next to the Lanczos and streaming solvers the
// reference still uses, so a maintainer would replace these seven function
// bodies with the calls below.  To run the reference's own acceptance suite
// (criterion 8, the approximation-operator algebra) against them WITHOUT
// editing the reference sources, oracle/Makefile links with -Wl,--wrap on each
// mangled name: the suite's calls land here, eigensolve.cpp stays as it is.
// Everything runs in fp64 (CURVKIT_F64): the suite holds 1e-10.
#include <cstdint>

#include "curv/eigensolve.hpp"
#include "curv/errors.hpp"
#include "curvkit_b200.h"

namespace curv {
namespace b200 {
void check(int rc);  // curvature_b200.cpp: curvkit status -> the reference's exceptions

namespace {
int64_t P(const EigenPairs& e) { return (int64_t)e.q.rows(); }
int64_t K(const EigenPairs& e) { return (int64_t)e.q.cols(); }

DenseMatrix materialize(const EigenPairs& e, int full, double lt, std::size_t cap) {
    const bool refuse = e.q.rows() > cap || (full && !(lt > 0.0));  // the library refuses before it writes
    DenseMatrix h(refuse ? 0 : e.q.rows(), refuse ? 0 : e.q.rows());
    check(curvkit_eig_materialize(P(e), K(e), e.q.data(), e.lambda.data(), full, lt, (int64_t)cap, CURVKIT_F64,
                                  h.data()));
    return h;
}

void apply(const EigenPairs& e, int full, double lt, const DenseVector& x, double* y, double* quad) {
    check(curvkit_eig_apply(P(e), K(e), e.q.data(), e.lambda.data(), full, lt, 1, x.data(), (int64_t)x.len(),
                            CURVKIT_F64, y, quad));
}
}  // namespace

void validate_eigen_pairs(const EigenPairs& e, double ortho_tol) {
    check(curvkit_eig_validate(P(e), K(e), e.q.data(), e.lambda.data(), (int64_t)e.lambda.len(), ortho_tol));
}

DenseMatrix low_rank_materialize(const EigenPairs& e, std::size_t cap) { return materialize(e, 0, 0.0, cap); }
DenseMatrix full_rank_materialize(const EigenPairs& e, double lt, std::size_t cap) { return materialize(e, 1, lt, cap); }

double low_rank_quadform(const EigenPairs& e, const DenseVector& x) {
    double q = 0.0;
    apply(e, 0, 0.0, x, nullptr, &q);
    return q;
}

double full_rank_quadform(const EigenPairs& e, double lt, const DenseVector& x) {
    double q = 0.0;
    apply(e, 1, lt, x, nullptr, &q);
    return q;
}

DenseVector low_rank_apply(const EigenPairs& e, const DenseVector& x) {
    DenseVector y(x.len() == e.q.rows() ? x.len() : 0);
    apply(e, 0, 0.0, x, y.data(), nullptr);
    return y;
}

DenseVector full_rank_apply(const EigenPairs& e, double lt, const DenseVector& x) {
    DenseVector y(x.len() == e.q.rows() && lt > 0.0 ? x.len() : 0);
    apply(e, 1, lt, x, y.data(), nullptr);
    return y;
}

}  // namespace b200
}  // namespace curv

// the --wrap targets (mangled names of the seven curv:: functions above)
#define CK_WRAP(sym) __wrap_##sym
extern "C" {
void CK_WRAP(_ZN4curv20validate_eigen_pairsERKNS_10EigenPairsEd)(const curv::EigenPairs& e, double tol) {
    curv::b200::validate_eigen_pairs(e, tol);
}
curv::DenseMatrix CK_WRAP(_ZN4curv20low_rank_materializeERKNS_10EigenPairsEm)(const curv::EigenPairs& e,
                                                                             std::size_t cap) {
    return curv::b200::low_rank_materialize(e, cap);
}
curv::DenseMatrix CK_WRAP(_ZN4curv21full_rank_materializeERKNS_10EigenPairsEdm)(const curv::EigenPairs& e, double lt,
                                                                               std::size_t cap) {
    return curv::b200::full_rank_materialize(e, lt, cap);
}
double CK_WRAP(_ZN4curv17low_rank_quadformERKNS_10EigenPairsERKNS_11DenseVectorE)(const curv::EigenPairs& e,
                                                                                 const curv::DenseVector& x) {
    return curv::b200::low_rank_quadform(e, x);
}
double CK_WRAP(_ZN4curv18full_rank_quadformERKNS_10EigenPairsEdRKNS_11DenseVectorE)(const curv::EigenPairs& e, double lt,
                                                                                   const curv::DenseVector& x) {
    return curv::b200::full_rank_quadform(e, lt, x);
}
curv::DenseVector CK_WRAP(_ZN4curv14low_rank_applyERKNS_10EigenPairsERKNS_11DenseVectorE)(const curv::EigenPairs& e,
                                                                                         const curv::DenseVector& x) {
    return curv::b200::low_rank_apply(e, x);
}
curv::DenseVector CK_WRAP(_ZN4curv15full_rank_applyERKNS_10EigenPairsEdRKNS_11DenseVectorE)(
    const curv::EigenPairs& e, double lt, const curv::DenseVector& x) {
    return curv::b200::full_rank_apply(e, lt, x);
}
}
