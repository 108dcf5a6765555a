// Sector-granular lane-recycling early-stop Monte-Carlo engine (block codes).
//
// The reference's early-stop campaign (harness.py:144-154 with
// SimulationConfig.early_stop, bp.py:242-256) decodes a batch until every
// lane's syndrome clears or the iteration cap is hit.  On a GPU that leaves
// straggler lanes scattered over every package: a 32-byte sector stays live
// while any of its 8 lanes is, so memory traffic barely drops.  Here lanes are
// recycled in groups of 8 (one sector): when all 8 codewords of a group have
// frozen (or hit the cap), the group immediately starts the next 8 codeword
// ids.  Fresh groups get their channel LLRs and beta^0 = mu written densely
// (sector-aligned) from a compact list, and the tuned check / variable passes
// run unchanged under the active-lane mask.  Each codeword still runs exactly
// the reference's early-stop schedule on its own lane (lanes never interact),
// so per-codeword results and the per-batch counters are identical; only the
// tick in which a codeword is decoded changes.
//
// Codeword id k of this rank is reference batch b = (k / gref) * W + rank,
// lane lane_base + b * gref + k % gref (batches round-robin over W ranks).
// Tick = fresh groups' channel + init -> check pass -> variable pass ->
// syndrome -> per-lane bit counts -> finish (count, freeze, reassign).
#include <cuda_runtime.h>

#include "block_kernels.cuh"
#include "philox.cuh"

namespace qcb {

int launch_vnu(const qc_plan* p, VnuArgs a, int mode, cudaStream_t s);
int launch_cnu_public(const qc_plan* p, CnuArgs a, int mode, cudaStream_t s);
int launch_syndrome_ext(const qc_plan* p, int gamma, const uint32_t* hb, uint32_t* bad, cudaStream_t s);


namespace {

constexpr int GROUP = 8;        // lanes per recycling group = one 32-byte sector of fp32

struct RcState {
  int64_t* slot_cw;        // (gamma) codeword id, -1 = none
  int32_t* slot_it;        // (gamma) iterations done
  int32_t* lane_bits;      // (gamma) hard-bit count of this tick
  int32_t* fresh_list;     // (gamma / GROUP) groups starting this tick
  int32_t* fresh_count;    // [1]
  uint32_t* active;        // (W) lanes still iterating
  uint32_t* bad;           // (W) syndrome failures of this tick
  uint32_t* fin;           // (W) lanes finishing this tick (frozen or capped)
  int64_t* next_group;     // [1] next group of codeword ids to hand out
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
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = g < c.gamma;
  const bool on = valid && g < c.id_limit;
  if (valid) {
    s.slot_cw[g] = on ? g : -1;
    s.slot_it[g] = 0;
    if (g % GROUP == 0) s.fresh_list[g / GROUP] = g / GROUP;
  }
  const unsigned w = __ballot_sync(0xffffffffu, on);
  if (valid && (g & 31) == 0) {
    s.active[g >> 5] = w;
    s.bad[g >> 5] = 0;
  }
  if (g == 0) {
    const int64_t groups = c.gamma / GROUP;
    const int64_t lim = (c.id_limit + GROUP - 1) / GROUP;
    *s.fresh_count = (int32_t)(groups < lim ? groups : lim);
    *s.next_group = groups;
  }
}

// channel LLRs of the fresh groups and their beta^0 = mu packages in phi form,
// in one pass: item = (fresh group, Philox block of 4 positions, lane in
// group).  Each (variable, lane) value is written to mu and to the J edges of
// the variable (QC arithmetic, codes.py:159-178); the 8 lanes of a group are
// consecutive threads, so every write fills whole 32-byte sectors.
__global__ void __launch_bounds__(THREADS) rc_fresh_kernel(RcState s, RcConfig c, const __grid_constant__ QcGrid grid,
                                                           float* mu, float* msgs, int n) {
  const int F = *s.fresh_count;
  const long long nblk = (n + 3) / 4;
  const long long items = (long long)F * nblk * GROUP;
  for (long long it = (long long)blockIdx.x * blockDim.x + threadIdx.x; it < items;
       it += (long long)gridDim.x * blockDim.x) {
    const int l = (int)(it % GROUP);
    const long long r = it / GROUP;
    const long long b = r % nblk;
    const int g = s.fresh_list[r / nblk] * GROUP + l;
    const int64_t k = s.slot_cw[g];
    if (k < 0) continue;
    uint64_t w[4];
    philox4x64_10((uint64_t)b + 1ull, ref_lane(c, k), 0ull, 0ull, c.k0, c.k1, w);
    const double s2 = __dmul_rn(c.sigma, c.sigma);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const long long pos = b * 4 + q;
      if (pos >= n) break;
      double y = __dadd_rn(1.0, __dmul_rn(c.sigma, ndtri_cephes(word_to_uniform(w[q]))));
      double m = __ddiv_rn(__dmul_rn(2.0, y), s2);
      m = m < -50.0 ? -50.0 : (m > 50.0 ? 50.0 : m);
      const float mf = __double2float_rn(m);
      mu[(size_t)pos * c.gamma + g] = mf;
      const float ps = __uint_as_float(__float_as_uint(psi_of_nat(fabsf(mf))) | (__float_as_uint(mf) & 0x80000000u));
      const int vb = div_p(grid, (int)pos), cc = (int)pos - vb * grid.p;
      for (int j = 0; j < grid.J; ++j) {
        int rr = cc - grid.s[j * grid.L + vb];
        rr += (rr < 0) ? grid.p : 0;
        msgs[((size_t)(j * grid.p + rr) * grid.L + vb) * c.gamma + g] = ps;
      }
    }
  }
}

// finish: count frozen / capped codewords, freeze them, restart finished groups
__global__ void rc_finish_kernel(RcState s, RcConfig c) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = g < c.gamma;
  const int64_t k = valid ? s.slot_cw[g] : -1;
  const bool was_active = valid && ((s.active[g >> 5] >> (g & 31)) & 1u);
  bool still = false;
  if (was_active) {
    const int it = s.slot_it[g] + 1;
    s.slot_it[g] = it;
    const bool ok = !((s.bad[g >> 5] >> (g & 31)) & 1u);
    if (ok || it >= c.max_it) {
      const int64_t b = (k / c.gref) * c.world + c.rank;
      if (b < c.n_batches) {
        const int bits = s.lane_bits[g];
        atomicAdd((unsigned long long*)&s.counts[b * 3 + 0], 1ull);
        atomicAdd((unsigned long long*)&s.counts[b * 3 + 1], (unsigned long long)bits);
        atomicAdd((unsigned long long*)&s.counts[b * 3 + 2], bits > 0 ? 1ull : 0ull);
      }
    } else {
      still = true;
    }
  }
  // a group restarts when none of its lanes is still iterating
  unsigned act = __ballot_sync(0xffffffffu, still);
  const int lane = g & 31, gl = lane & ~(GROUP - 1);
  const bool group_idle = ((act >> gl) & 0xffu) == 0;
  bool start = false;
  int64_t ng = 0;
  if (valid && group_idle && (g % GROUP) == 0) ng = (int64_t)atomicAdd((unsigned long long*)s.next_group, 1ull);
  ng = __shfl_sync(0xffffffffu, ng, gl);          // the group leader's new group id
  if (valid && group_idle) {
    const int64_t nk = ng * GROUP + (g % GROUP);
    start = nk < c.id_limit;
    s.slot_cw[g] = start ? nk : -1;
    s.slot_it[g] = 0;
    if (start && (g % GROUP) == 0) s.fresh_list[atomicAdd(s.fresh_count, 1)] = g / GROUP;
  }
  act = __ballot_sync(0xffffffffu, still || start);
  if (valid && lane == 0) {
    s.active[g >> 5] = act;
    s.bad[g >> 5] = 0;
  }
}

__global__ void rc_reset_fresh_kernel(int32_t* fresh_count) { *fresh_count = 0; }

// lanes that finish this tick (syndrome clean or at the iteration cap): the
// only ones whose bit errors are counted (rc_finish_kernel)
__global__ void rc_fin_mask_kernel(RcState s, RcConfig c) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = g < c.gamma;
  bool f = false;
  if (valid && ((s.active[g >> 5] >> (g & 31)) & 1u))
    f = !((s.bad[g >> 5] >> (g & 31)) & 1u) || s.slot_it[g] + 1 >= c.max_it;
  const unsigned m = __ballot_sync(0xffffffffu, f);
  if (valid && (g & 31) == 0) s.fin[g >> 5] = m;
}

}  // namespace
}  // namespace qcb

using namespace qcb;

namespace {
RcState rc_state(void* base, int gamma) {
  const size_t W = (size_t)gamma / 32;
  char* p = static_cast<char*>(base);
  RcState s;
  s.slot_cw = reinterpret_cast<int64_t*>(p); p += (size_t)gamma * 8;
  s.next_group = reinterpret_cast<int64_t*>(p); p += 8;
  s.slot_it = reinterpret_cast<int32_t*>(p); p += (size_t)gamma * 4;
  s.lane_bits = reinterpret_cast<int32_t*>(p); p += (size_t)gamma * 4;
  s.fresh_list = reinterpret_cast<int32_t*>(p); p += (size_t)(gamma / GROUP) * 4;
  s.fresh_count = reinterpret_cast<int32_t*>(p); p += 8;
  s.active = reinterpret_cast<uint32_t*>(p); p += W * 4;
  s.bad = reinterpret_cast<uint32_t*>(p); p += W * 4;
  s.fin = reinterpret_cast<uint32_t*>(p);
  s.counts = nullptr;
  return s;
}
}  // namespace

extern "C" {

size_t qc_rc_state_bytes(int gamma) {
  const size_t G = (size_t)(gamma > 0 ? gamma : 0);
  return G * 8 + 8 + G * 4 + G * 4 + (G / GROUP) * 4 + 8 + 3 * (G / 32) * 4 + 64;
}

int qc_rc_init(int gamma, int64_t id_limit, void* state, void* stream) {
  if (gamma <= 0 || gamma % 128 || !state) return fail_arg("bad recycling state arguments");
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
  if (gamma <= 0 || gamma % 128 || gamma_ref <= 0 || world < 1 || rank < 0 || rank >= world || max_it < 1 ||
      ticks < 0)
    return fail_arg("bad recycling arguments");
  if (!p->qc_regular) return fail_arg("lane recycling needs an all-live QC grid");
  cudaStream_t st = as_stream(stream);
  RcState s = rc_state(state, gamma);
  s.counts = counts;
  RcConfig c{gamma, gamma_ref, world, rank, max_it, id_limit, n_batches, seed_lo, seed_hi, lane_base, sigma};
  const QcGrid g = make_grid(p);
  static int nsm = 0;
  if (!nsm) {
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  const unsigned persist = (unsigned)nsm * (2048 / THREADS);   // 2048 threads per SM
  int rc;
  for (int t = 0; t < ticks; ++t) {
    rc_fresh_kernel<<<persist, THREADS, 0, st>>>(s, c, g, mu, msgs, p->N);
    rc_reset_fresh_kernel<<<1, 1, 0, st>>>(s.fresh_count);
    CnuArgs a{msgs, mu, p->d_check_ptr, p->d_edge_var, s.active, nullptr, p->M, gamma};
    if ((rc = launch_cnu_public(p, a, CNU_PHI, st))) return rc;
    VnuArgs v{};
    v.msgs = msgs; v.mu = mu; v.hb = hb; v.active = s.active; v.gamma = gamma;
    if ((rc = launch_vnu(p, v, VNU_PHI, st))) return rc;
    if ((rc = launch_syndrome_ext(p, gamma, hb, s.bad, st))) return rc;
    rc_fin_mask_kernel<<<blocks_for(gamma), THREADS, 0, st>>>(s, c);
    if ((rc = launch_bit_errors_ext(p, gamma, hb, s.lane_bits, st, s.fin))) return rc;
    rc_finish_kernel<<<blocks_for(gamma), THREADS, 0, st>>>(s, c);
  }
  return check_launch("qc_rc_ticks");
}

/* host-readable progress: next group id (int64) */
int qc_rc_next_id(int gamma, const void* state, int64_t* next_id_dev_out, void* stream) {
  if (!state || !next_id_dev_out) return fail_arg("null argument");
  const RcState s = rc_state(const_cast<void*>(state), gamma);
  cudaMemcpyAsync(next_id_dev_out, s.next_group, 8, cudaMemcpyDeviceToDevice, as_stream(stream));
  return check_launch("qc_rc_next_id");
}

}  // extern "C"
