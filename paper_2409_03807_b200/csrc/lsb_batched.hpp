// Batched (many-z) evaluation, subspace Hessians and the second-order
// Lipschitz loss (SURVEY §2.2 kernels K7-K9).
#pragma once

#include "lsb_context.hpp"

namespace lsb {

void batched_eval(Context& c, int B, const double* Z, double* E, double* G);
void batched_hessian(Context& c, int B, const double* Z, double* H);
void batched_objective_hessian(Context& c, int B, const double* Z, double* H);
double lipschitz_loss(Context& c, int P, const double* Z1, const double* Z2);
double lipschitz_loss_grad(Context& c, int P, const double* Z1, const double* Z2, double* grad);

}  // namespace lsb
