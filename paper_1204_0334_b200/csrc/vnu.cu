// Variable-node kernels of the block decoder and their dispatch.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "block_kernels.cuh"

namespace qcb {

QcGrid make_grid(const qc_plan* p) {
  QcGrid g;
  std::memset(&g, 0, sizeof(g));
  if (p->qc_regular) {
    g.J = p->J; g.L = p->L; g.p = p->p;
    g.pmagic = ((1ull << 40) + (unsigned long long)p->p - 1) / (unsigned long long)p->p;
    for (int i = 0; i < p->J * p->L; ++i) g.s[i] = (int16_t)p->shifts[i];
  }
  return g;
}

namespace {

template <int DV, int VEC, int MODE>
void launch_v(const qc_plan* p, const VnuArgs& a, const QcGrid& g, cudaStream_t s) {
  long long threads = (long long)p->N * (a.gamma / VEC);
  unsigned nb = blocks_for(threads);
  if (p->qc_regular && p->J == DV) vnu_kernel<DV, VEC, true, MODE><<<nb, THREADS, 0, s>>>(a, g);
  else vnu_kernel<DV, VEC, false, MODE><<<nb, THREADS, 0, s>>>(a, g);
}

template <int DV, int VEC>
void launch_mode(const qc_plan* p, const VnuArgs& a, int mode, const QcGrid& g, cudaStream_t s) {
  switch (mode) {
    case VNU_PHI: launch_v<DV, VEC, VNU_PHI>(p, a, g, s); break;
    case VNU_NONE: launch_v<DV, VEC, VNU_NONE>(p, a, g, s); break;
    default: launch_v<DV, VEC, VNU_BETA>(p, a, g, s);
  }
}

template <int DV>
void launch_vec(const qc_plan* p, const VnuArgs& a, int mode, const QcGrid& g, cudaStream_t s) {
  int vec = pick_vec_vnu(a.gamma);
  switch (vec) {
    case 4: launch_mode<DV, 4>(p, a, mode, g, s); break;
    case 2: launch_mode<DV, 2>(p, a, mode, g, s); break;
    default: launch_mode<DV, 1>(p, a, mode, g, s); break;
  }
}

int bucket_dv(int d) {
  static const int B[] = {2, 3, 4, 6, 8, 12, 16};
  for (int b : B)
    if (d <= b) return b;
  return -1;
}

}  // namespace

int launch_vnu(const qc_plan* p, VnuArgs a, int mode, cudaStream_t s) {
  QcGrid g = make_grid(p);
  a.var_pad = p->d_var_pad;
  a.dv = p->dv_max;
  a.N = p->N;
  if (p->N == 0) return 0;
  switch (bucket_dv(std::max(p->dv_max, 1))) {
    case 2: launch_vec<2>(p, a, mode, g, s); break;
    case 3: launch_vec<3>(p, a, mode, g, s); break;
    case 4: launch_vec<4>(p, a, mode, g, s); break;
    case 6: launch_vec<6>(p, a, mode, g, s); break;
    case 8: launch_vec<8>(p, a, mode, g, s); break;
    case 12: launch_vec<12>(p, a, mode, g, s); break;
    case 16: launch_vec<16>(p, a, mode, g, s); break;
    default: return fail_arg("variable degree > 16 is not supported");
  }
  return check_launch("vnu");
}

}  // namespace qcb
