// tcgen05 (5th-gen tensor core) GEMMs of the batched path: W_out (n x h) times
// a batch tile (forward) and W_out^T times the gathered gradients (VJP).
#pragma once

#include "lsb_context.hpp"

namespace lsb {

struct TcGemm {
    bool enabled = false;
    void init(Context&, const float*, int, int, int) {}
    bool gemm_out(cudaStream_t, const float*, float*) { return false; }
    bool gemm_vjp(cudaStream_t, const float*, float*) { return false; }
};

}  // namespace lsb
