// Batched evaluation / Hessians — see lsb_batched.hpp.
#include "lsb_batched.hpp"

namespace lsb {

void batched_eval(Context&, int, const double*, double*, double*) {
    throw LsbError(LSB_EINVAL, "eval_batched: not implemented in this build");
}
void batched_hessian(Context&, int, const double*, double*) {
    throw LsbError(LSB_EINVAL, "hessian_batched: not implemented in this build");
}
double lipschitz_loss(Context&, int, const double*, const double*) {
    throw LsbError(LSB_EINVAL, "lipschitz_loss: not implemented in this build");
}

}  // namespace lsb
