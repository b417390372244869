// Translation unit of the lower-level QP kernel, compiled with FMA
// contraction (see qp.cuh). engine.cu launches it through launch_qp_kernel.
#include "qp.cuh"

namespace gdev {

void launch_qp_kernel(const DevHand& H, const DevParams& P, const DevState& st, int m, int mode, int with_grad,
                      cudaStream_t stream) {
  const unsigned blocks = static_cast<unsigned>((st.G + GDEV_QP_WARPS - 1) / GDEV_QP_WARPS);
  constexpr int kThreads = 32 * GDEV_QP_WARPS;
  if (P.k == 8) {
    switch (m) {
      case 1: k_qp_t<8, 1><<<blocks, kThreads, 0, stream>>>(H, P, st, m, mode, with_grad); return;
      case 2: k_qp_t<8, 2><<<blocks, kThreads, 0, stream>>>(H, P, st, m, mode, with_grad); return;
      case 3: k_qp_t<8, 3><<<blocks, kThreads, 0, stream>>>(H, P, st, m, mode, with_grad); return;
      case 4: k_qp_t<8, 4><<<blocks, kThreads, 0, stream>>>(H, P, st, m, mode, with_grad); return;
      case 5: k_qp_t<8, 5><<<blocks, kThreads, 0, stream>>>(H, P, st, m, mode, with_grad); return;
      default: break;
    }
  }
  k_qp_t<0, 0><<<blocks, kThreads, 0, stream>>>(H, P, st, m, mode, with_grad);
}

}  // namespace gdev
