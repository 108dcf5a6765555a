// Host-side launcher of the check-node kernels for one degree bucket DC.
#pragma once

#include "block_kernels.cuh"

namespace qcb {

template <int DC, int VEC>
int launch_cnu_v(const qc_plan* p, const CnuArgs& a, int mode, cudaStream_t s) {
  long long threads = (long long)p->M * (a.gamma / VEC);
  unsigned nb = blocks_for(threads);
  const QcGrid g = make_grid(p);
  const bool reg = p->check_regular == DC;
  const bool qc = p->qc_regular;
  switch (mode) {
    case CNU_FROM_MU:
      if (qc && reg) cnu_kernel<DC, VEC, true, CNU_FROM_MU, true><<<nb, THREADS, 0, s>>>(a, g);
      else if (reg) cnu_kernel<DC, VEC, true, CNU_FROM_MU, false><<<nb, THREADS, 0, s>>>(a, g);
      else cnu_kernel<DC, VEC, false, CNU_FROM_MU, false><<<nb, THREADS, 0, s>>>(a, g);
      break;
    case CNU_PHI:
      if (reg) cnu_kernel<DC, VEC, true, CNU_PHI, false><<<nb, THREADS, 0, s>>>(a, g);
      else cnu_kernel<DC, VEC, false, CNU_PHI, false><<<nb, THREADS, 0, s>>>(a, g);
      break;
    default:
      if (reg) cnu_kernel<DC, VEC, true, CNU_BETA, false><<<nb, THREADS, 0, s>>>(a, g);
      else cnu_kernel<DC, VEC, false, CNU_BETA, false><<<nb, THREADS, 0, s>>>(a, g);
  }
  return 0;
}

template <int DC>
int launch_cnu_dc(const qc_plan* p, const CnuArgs& a, int mode, cudaStream_t s) {
  switch (pick_vec_cnu(a.gamma, DC)) {
    case 2: return launch_cnu_v<DC, 2>(p, a, mode, s);
    default: return launch_cnu_v<DC, 1>(p, a, mode, s);
  }
}

}  // namespace qcb
