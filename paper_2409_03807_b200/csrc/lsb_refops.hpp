// Device versions of the reference's secondary hot-path primitives (lsb_refops.cu).
#pragma once

#include "lsb_context.hpp"

namespace lsb {

void refops_assemble(Context& c, const double* q, double* value, double* grad);
void refops_elastic_hessian_apply(Context& c, const double* q, int k, const double* in, double* out);
void refops_element_snh(Context& c, int count, const int* ids, const double* positions, double* energy,
                        double* grad, double* hess);
void refops_decode_jacobian(Context& c, const double* z, double* J);
void refops_decode_second_directional(Context& c, const double* z, const double* u, const double* v, double* out);

}  // namespace lsb
