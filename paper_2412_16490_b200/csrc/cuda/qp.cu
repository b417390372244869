// Translation unit of the lower-level QP kernel, compiled with FMA
// contraction (see qp.cuh). engine.cu launches it through launch_qp_kernel.
#include "qp.cuh"

namespace gdev {

void launch_qp_kernel(const DevHand& H, const DevParams& P, const DevState& st, int m, int mode, int with_grad,
                      cudaStream_t stream) {
  const unsigned blocks = static_cast<unsigned>((st.G + 3) / 4);
  k_qp<<<blocks, 128, 0, stream>>>(H, P, st, m, mode, with_grad);
}

}  // namespace gdev
