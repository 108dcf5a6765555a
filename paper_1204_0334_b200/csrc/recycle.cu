// Lane-recycling early-stop Monte-Carlo engine for regular QC block codes.
//
// The reference's early-stop campaign (harness.py:144-154 with
// SimulationConfig.early_stop, bp.py:242-256) decodes each batch of gamma
// codewords until every lane's syndrome clears or the iteration cap is hit;
// on a GPU that leaves the late, sparse lanes scattered over every package, so
// the memory traffic barely drops.  Here a lane ("slot") whose codeword has
// frozen immediately takes the next codeword id and restarts from its channel
// LLRs, so every tick (one flooding iteration of all slots) does dense work.
// Each codeword still runs exactly the reference's early-stop schedule on its
// own lane (lanes never interact), so per-codeword bits / errors and therefore
// the per-batch counters are identical; only the tick in which a codeword is
// decoded changes.
//
// Codeword id k of this rank maps to reference batch b = (k / gref) * W + rank
// and lane lane_base + b * gref + k % gref (batches round-robin over W ranks).
// Per tick: channel (fresh slots) -> check pass (fresh slots read mu) ->
// variable pass (phi form + hard-bit planes) -> syndrome -> per-slot bit
// counts -> finish (count, reassign).
#include <cuda_runtime.h>

#include "block_kernels.cuh"
#include "philox.cuh"

namespace qcb {
namespace {

struct RcState {
  int64_t* slot_cw;        // (gamma) codeword id or -1
  int32_t* slot_it;        // (gamma) iterations done
  uint32_t* fresh;         // (W) slots that start a codeword this tick
  uint32_t* active;        // (W) slots holding a codeword
  uint32_t* bad;           // (W) syndrome failures of this tick
  int32_t* lane_bits;      // (gamma) hard-bit count of this tick
  int64_t* next_id;        // [1] next codeword id to hand out
  int64_t* counts;         // (n_batches, 3) frames, bit errors, frame errors
};

struct RcConfig {
  int gamma, gref, world, rank, max_it;
  int64_t id_limit;        // codeword ids >= id_limit are not started
  int64_t n_batches;       // rows of counts
  uint64_t k0, k1, lane_base;
  double sigma;
};

__device__ __forceinline__ uint64_t ref_lane(const RcConfig& c, int64_t k) {
  const int64_t b = (k / c.gref) * c.world + c.rank;
  return c.lane_base + (uint64_t)(b * c.gref + k % c.gref);
}

__global__ void rc_init_kernel(RcState s, RcConfig c) {
  int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g < c.gamma) {
    int64_t k = g < c.id_limit ? g : -1;
    s.slot_cw[g] = k;
    s.slot_it[g] = 0;
  }
  if (g < c.gamma / 32) {
    uint32_t on = 0;
    for (int b = 0; b < 32; ++b)
      if (g * 32 + b < c.id_limit) on |= 1u << b;
    s.fresh[g] = on;
    s.active[g] = on;
    s.bad[g] = 0;
  }
  if (g == 0) *s.next_id = c.gamma < c.id_limit ? c.gamma : c.id_limit;
}

// channel LLRs of fresh slots only (thread = (slot g, Philox block of 4 positions))
__global__ void __launch_bounds__(THREADS) rc_channel_kernel(RcState s, RcConfig c, float* mu, int n) {
  long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nblk = (n + 3) / 4;
  if (tid >= nblk * c.gamma) return;
  const int g = (int)(tid % c.gamma);
  if (!((s.fresh[g >> 5] >> (g & 31)) & 1u)) return;
  const long long b = tid / c.gamma;
  uint64_t w[4];
  philox4x64_10((uint64_t)b + 1ull, ref_lane(c, s.slot_cw[g]), 0ull, 0ull, c.k0, c.k1, w);
  const double s2 = __dmul_rn(c.sigma, c.sigma);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const long long pos = b * 4 + k;
    if (pos >= n) break;
    double y = __dadd_rn(1.0, __dmul_rn(c.sigma, ndtri_cephes(word_to_uniform(w[k]))));
    double m = __ddiv_rn(__dmul_rn(2.0, y), s2);
    m = m < -50.0 ? -50.0 : (m > 50.0 ? 50.0 : m);
    mu[(size_t)pos * c.gamma + g] = __double2float_rn(m);
  }
}

// check pass, phi form; fresh lanes take beta^0 = mu (fused init), idle lanes skip
template <int DC, int VEC>
__global__ void __launch_bounds__(THREADS) rc_cnu_kernel(CnuArgs a, const __grid_constant__ QcGrid grid,
                                                        const uint32_t* fresh) {
  const int GV = a.gamma / VEC;
  long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (long long)a.M * GV) return;
  int m = (int)(tid / GV), q = (int)(tid - (long long)m * GV);
  const unsigned lanes = lane_bits_of(a.active, q * VEC, VEC);
  if (lanes == 0) return;
  const unsigned fr = lane_bits_of(fresh, q * VEC, VEC) & lanes;
  const int e0 = m * DC;
  float x[DC][VEC];
#pragma unroll
  for (int k = 0; k < DC; ++k) vload<VEC>(a.msgs + (size_t)(e0 + k) * a.gamma + q * VEC, x[k]);
  if (fr) {
    const int jrow = m / grid.p, r = m - jrow * grid.p;
#pragma unroll
    for (int k = 0; k < DC; ++k) {
      int c = r + grid.s[jrow * grid.L + k];
      c -= (c >= grid.p) ? grid.p : 0;
      float mv[VEC];
      vload<VEC>(a.mu + (size_t)(k * grid.p + c) * a.gamma + q * VEC, mv);
#pragma unroll
      for (int i = 0; i < VEC; ++i)
        if ((fr >> i) & 1u)
          x[k][i] = __uint_as_float(__float_as_uint(psi_of_nat(fabsf(mv[i]))) |
                                    (__float_as_uint(mv[i]) & 0x80000000u));
    }
  }
  cnu_core<DC, VEC, true>(x, DC, lanes);
#pragma unroll
  for (int k = 0; k < DC; ++k) vstore<VEC>(a.msgs + (size_t)(e0 + k) * a.gamma + q * VEC, x[k]);
}

// finish: count frozen / capped codewords into their batch, hand out new ids
__global__ void rc_finish_kernel(RcState s, RcConfig c) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = g < c.gamma;
  const int64_t k = valid ? s.slot_cw[g] : -1;
  bool start = false;
  if (k >= 0) {
    const int it = s.slot_it[g] + 1;
    const bool ok = !((s.bad[g >> 5] >> (g & 31)) & 1u);
    if (ok || it >= c.max_it) {
      const int64_t b = (k / c.gref) * c.world + c.rank;
      if (b < c.n_batches) {
        const int bits = s.lane_bits[g];
        atomicAdd((unsigned long long*)&s.counts[b * 3 + 0], 1ull);
        atomicAdd((unsigned long long*)&s.counts[b * 3 + 1], (unsigned long long)bits);
        atomicAdd((unsigned long long*)&s.counts[b * 3 + 2], bits > 0 ? 1ull : 0ull);
      }
      const int64_t nk = (int64_t)atomicAdd((unsigned long long*)s.next_id, 1ull);
      if (nk < c.id_limit) {
        s.slot_cw[g] = nk;
        s.slot_it[g] = 0;
        start = true;
      } else {
        s.slot_cw[g] = -1;
      }
    } else {
      s.slot_it[g] = it;
    }
  }
  // rebuild the 32-lane words (one warp = one word: gamma % 32 == 0)
  const unsigned fw = __ballot_sync(0xffffffffu, start);
  const unsigned aw = __ballot_sync(0xffffffffu, valid && s.slot_cw[valid ? g : 0] >= 0);
  if (valid && (g & 31) == 0) {
    s.fresh[g >> 5] = fw;
    s.active[g >> 5] = aw;
    s.bad[g >> 5] = 0;
  }
}

int launch_rc_cnu(const qc_plan* p, const CnuArgs& a, const QcGrid& g, const uint32_t* fresh, cudaStream_t st) {
  if (!p->qc_regular || p->check_regular != 24) return fail_arg("lane recycling needs a regular (J, 24) QC grid");
  if (a.gamma % 64) return fail_arg("lane recycling needs gamma % 64 == 0");
  const long long n = (long long)p->M * (a.gamma / 2);
  rc_cnu_kernel<24, 2><<<blocks_for(n), THREADS, 0, st>>>(a, g, fresh);
  return check_launch("rc_cnu");
}

}  // namespace

int launch_vnu(const qc_plan* p, VnuArgs a, int mode, cudaStream_t s);
int launch_syndrome_ext(const qc_plan* p, int gamma, const uint32_t* hb, uint32_t* bad, cudaStream_t s);
int launch_bit_errors_ext(const qc_plan* p, int gamma, const uint32_t* hb, int32_t* lane_bits, cudaStream_t s);

}  // namespace qcb

using namespace qcb;

extern "C" {

size_t qc_rc_state_bytes(int gamma) {
  const size_t W = (size_t)(gamma > 0 ? gamma : 0) / 32;
  return gamma * 8 + gamma * 4 + 3 * W * 4 + gamma * 4 + 8 + 64;
}

static RcState rc_state(void* base, int gamma) {
  const size_t W = (size_t)gamma / 32;
  char* p = static_cast<char*>(base);
  RcState s;
  s.slot_cw = reinterpret_cast<int64_t*>(p); p += (size_t)gamma * 8;
  s.next_id = reinterpret_cast<int64_t*>(p); p += 8;
  s.slot_it = reinterpret_cast<int32_t*>(p); p += (size_t)gamma * 4;
  s.lane_bits = reinterpret_cast<int32_t*>(p); p += (size_t)gamma * 4;
  s.fresh = reinterpret_cast<uint32_t*>(p); p += W * 4;
  s.active = reinterpret_cast<uint32_t*>(p); p += W * 4;
  s.bad = reinterpret_cast<uint32_t*>(p);
  s.counts = nullptr;
  return s;
}

int qc_rc_init(int gamma, int64_t id_limit, void* state, void* stream) {
  if (gamma <= 0 || gamma % 64 || !state) return fail_arg("bad recycling state arguments");
  RcState s = rc_state(state, gamma);
  RcConfig c{};
  c.gamma = gamma;
  c.id_limit = id_limit;
  rc_init_kernel<<<blocks_for(gamma), THREADS, 0, as_stream(stream)>>>(s, c);
  return check_launch("qc_rc_init");
}

int qc_rc_ticks(const qc_plan* p, int gamma, int gamma_ref, int world, int rank, int max_it, int64_t id_limit,
                int64_t n_batches, uint64_t seed_lo, uint64_t seed_hi, uint64_t lane_base, double sigma, int ticks,
                float* mu, float* msgs, uint32_t* hb, void* state, int64_t* counts, void* stream) {
  if (!p || !mu || !msgs || !hb || !state || !counts) return fail_arg("null argument");
  if (gamma <= 0 || gamma % 64 || gamma_ref <= 0 || world < 1 || rank < 0 || rank >= world || max_it < 1 || ticks < 0)
    return fail_arg("bad recycling arguments");
  cudaStream_t st = as_stream(stream);
  RcState s = rc_state(state, gamma);
  s.counts = counts;
  RcConfig c{gamma, gamma_ref, world, rank, max_it, id_limit, n_batches, seed_lo, seed_hi, lane_base, sigma};
  const QcGrid g = make_grid(p);
  int rc;
  for (int t = 0; t < ticks; ++t) {
    const long long nch = (long long)((p->N + 3) / 4) * gamma;
    rc_channel_kernel<<<blocks_for(nch), THREADS, 0, st>>>(s, c, mu, p->N);
    CnuArgs a{msgs, mu, p->d_check_ptr, p->d_edge_var, s.active, nullptr, p->M, gamma};
    if ((rc = launch_rc_cnu(p, a, g, s.fresh, st))) return rc;
    VnuArgs v{};
    v.msgs = msgs; v.mu = mu; v.hb = hb; v.active = s.active; v.gamma = gamma;
    if ((rc = launch_vnu(p, v, VNU_PHI, st))) return rc;
    if ((rc = launch_syndrome_ext(p, gamma, hb, s.bad, st))) return rc;
    if ((rc = launch_bit_errors_ext(p, gamma, hb, s.lane_bits, st))) return rc;
    rc_finish_kernel<<<blocks_for(gamma), THREADS, 0, st>>>(s, c);
  }
  return check_launch("qc_rc_ticks");
}

/* host-readable progress: next_id (int64) */
int qc_rc_next_id(int gamma, const void* state, int64_t* next_id_dev_out, void* stream) {
  if (!state || !next_id_dev_out) return fail_arg("null argument");
  const RcState s = rc_state(const_cast<void*>(state), gamma);
  cudaMemcpyAsync(next_id_dev_out, s.next_id, 8, cudaMemcpyDeviceToDevice, as_stream(stream));
  return check_launch("qc_rc_next_id");
}

}  // extern "C"
