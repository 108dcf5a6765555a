/*
 * qcldpc_b200 -- C ABI of the B200-native LDPC / LDPCCC belief-propagation path.
 *
 * Every entry point replaces one numpy function of the reference package
 * (/root/reference/pkg/src/qcldpc); the cited file:line is the interface it
 * stands in for.  The Python host layer (paper_1204_0334_b200/_lib.py) binds
 * these with ctypes; INTEGRATION.md shows the binding a maintainer of the
 * reference would add.
 *
 * Conventions
 *  - All array arguments are caller-owned DEVICE pointers (e.g. torch tensors),
 *    except the host-side plan inputs of qc_plan_create_* (HOST pointers).
 *  - gamma (lanes per batch, "Gamma" in the paper) must be a positive multiple
 *    of 32; callers pad.  Lane g of a 32-lane word is bit (g & 31) of word g>>5.
 *  - Message store: edge-major (E, gamma) fp32, edge ids row-major as in
 *    codes.py:181-257.  Channel LLRs / posteriors: variable-major (N, gamma).
 *    Hard-bit planes: (N, gamma/32) uint32.
 *  - stream: a cudaStream_t passed as void*; 0 = legacy default stream.
 *  - Return value: 0 ok; < 0 argument error (ValueError class); > 0 runtime /
 *    CUDA error (RuntimeError class).  qc_last_error() gives the thread-local
 *    message of the last failure.
 *  - Plans are immutable after creation and safe to share across threads.
 */
#ifndef QCLDPC_B200_H
#define QCLDPC_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define QC_API __attribute__((visibility("default")))
#else
#define QC_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct qc_plan qc_plan;
typedef struct cc_plan cc_plan;

/* ---- errors / info ------------------------------------------------------ */
QC_API const char* qc_last_error(void);
QC_API int qc_abi_version(void);

/* ---- code plans (replaces EdgeLayout/build_edge_layout, codes.py:181-257) */
/* QC grid (J x L shifts, -1 = zero block), host pointer; replaces
 * expand_qc + build_edge_layout (codes.py:159-178, 224-257). */
QC_API int qc_plan_create_qc(const int64_t* shifts, int J, int L, int p, qc_plan** out);
/* Arbitrary sparse H in the reference's row-major edge numbering:
 * check_ptr (M+1), edge_var (E) -- EdgeLayout.check_ptr / .edge_var. */
QC_API int qc_plan_create_csr(int n_vars, int n_checks, const int64_t* check_ptr,
                       const int64_t* edge_var, qc_plan** out);
QC_API void qc_plan_destroy(qc_plan* plan);
/* dims[0..5] = N, M, E, dc_max, dv_max, check_regular (0 if irregular) */
QC_API int qc_plan_dims(const qc_plan* plan, int64_t* dims);

/* ---- block decoder kernels (bp.py) -------------------------------------- */
/* MessageBatch.__init__ (bp.py:74-84): msgs[e] = mu[edge_var[e]]. */
QC_API int qc_init(const qc_plan* plan, int gamma, const float* mu, float* msgs, void* stream);
/* check_node_update (bp.py:134-162), in place; active = (gamma/32) lane-mask
 * words or NULL (all lanes). */
QC_API int qc_cnu(const qc_plan* plan, int gamma, float* msgs, const uint32_t* active,
           void* stream);
/* variable_node_update (bp.py:165-188): msgs <- beta on active lanes (frozen
 * lanes keep their packages, bp.py:185-186), post (N,gamma) <- clip(total) on
 * EVERY lane (bp.py:183; post may be NULL); hb (N,gamma/32) hard-bit planes of
 * post (may be NULL). */
QC_API int qc_vnu(const qc_plan* plan, int gamma, float* msgs, const float* mu, float* post,
           uint32_t* hb, const uint32_t* active, void* stream);
/* The same passes in the representation used inside qc_decode:
 * cnu mode 0 = beta in (qc_cnu), 1 = beta^0 gathered from mu (fused init),
 * 2 = var->check packages hold sign(beta)*phi(|beta|) ("phi form");
 * vnu mode 0 = write beta (qc_vnu), 1 = write phi form, 2 = no message write. */
QC_API int qc_cnu_ex(const qc_plan* plan, int gamma, int mode, float* msgs, const float* mu,
                     const uint32_t* active, void* stream);
QC_API int qc_vnu_ex(const qc_plan* plan, int gamma, int mode, float* msgs, const float* mu,
                     float* post, uint32_t* hb, const uint32_t* active, void* stream);
/* hard_decision_and_syndrome (bp.py:191-210) on hard-bit planes:
 * bad[w] |= lanes of word w with an odd check (bad must be zeroed by caller). */
QC_API int qc_syndrome(const qc_plan* plan, int gamma, const uint32_t* hb, uint32_t* bad,
                void* stream);
/* posterior -> hard-bit planes (bits = post < 0) */
QC_API int qc_hard_bits(const qc_plan* plan, int gamma, const float* post, uint32_t* hb, void* stream);
/* per-lane count of set hard bits (all-zero codeword => bit errors) */
QC_API int qc_bit_errors(const qc_plan* plan, int gamma, const uint32_t* hb, int32_t* lane_bits,
                  void* stream);

/* decode_llr_batch (bp.py:213-265), whole loop on device.
 * mu (N,gamma) clipped LLRs; msgs (E,gamma) scratch; post (N,gamma) out;
 * hb (N,gamma/32) out; work: qc_decode_work_words(plan, gamma) uint32 scratch
 * (for regular QC codes it holds the compact check records, 3 M gamma words);
 * ok (gamma) u8 out; iters_run (gamma) i32 out; lane_bits (gamma) i32 out
 * (may be NULL).  early_stop reproduces bp.py:242-256 (freeze on syndrome). */
QC_API size_t qc_decode_work_words(const qc_plan* plan, int gamma);
/* word offset of the compact check records inside that work buffer (for the
 * qc_agg_* pass entry points used by benchmarks and tests). */
QC_API size_t qc_decode_records_offset(int gamma);
QC_API int qc_decode(const qc_plan* plan, int gamma, int iters, int early_stop, const float* mu,
              float* msgs, float* post, uint32_t* hb, uint32_t* work, uint8_t* ok,
              int32_t* iters_run, int32_t* lane_bits, void* stream);

/* The two passes of qc_decode's compact check-state schedule (regular QC
 * plans; bit-identical to qc_cnu_ex mode 2 + qc_vnu_ex mode 1):
 * qc_agg_check: check records agg (M, 3, gamma) = (S | parity sign bit, S2, max)
 *   of the phi-form packages (from_mu = 1: of beta^0 = mu, iteration 1);
 * qc_agg_var: each variable re-derives its check->var messages from agg and the
 *   package it replaces (flags & 1: iteration 1, packages implied by mu), then
 *   writes phi-form packages, or (flags & 2: last iteration) post / hb only. */
QC_API int qc_agg_check(const qc_plan* plan, int gamma, int from_mu, float* msgs, const float* mu,
                        float* agg, void* stream);
QC_API int qc_agg_var(const qc_plan* plan, int gamma, int flags, float* msgs, const float* mu,
                      const float* agg, float* post, uint32_t* hb, void* stream);
/* One launch of both: qc_agg_var on lanes [var_lane0, +lanes) and qc_agg_check
 * on lanes [check_lane0, +lanes) (disjoint windows, 128-lane aligned, gamma %
 * 256 == 0; the decode loop's half-iteration step). */
QC_API int qc_agg_fused(const qc_plan* plan, int gamma, int lanes, int var_lane0, int var_flags,
                        int check_lane0, int check_from_mu, float* msgs, const float* mu, float* agg,
                        float* post, uint32_t* hb, void* stream);
/* kernels qc_decode launches for these arguments (bench accounting) */
QC_API int qc_decode_launches(const qc_plan* plan, int gamma, int iters, int early_stop);
/* decode_llr_batch(..., early_stop=True) with lane compaction (bp.py:242-256):
 * at a few checkpoint iterations the lanes still iterating are packed into a
 * second buffer set, so converged lanes stop costing work; results equal
 * qc_decode(early_stop = 1) bit for bit (posteriors, bits, ok, iterations_run).
 * scratch: qc_decode_es_scratch_words(plan, gamma) 32-bit words of device
 * memory (0 = plan / gamma / iterations not eligible: falls back to qc_decode).
 * Other arguments as qc_decode. */
QC_API int qc_decode_es(const qc_plan* plan, int gamma, int iters, const float* mu, float* msgs, float* post,
                        uint32_t* hb, uint32_t* work, uint32_t* scratch, uint8_t* ok, int32_t* iters_run,
                        int32_t* lane_bits, void* stream);
QC_API size_t qc_decode_es_scratch_words(const qc_plan* plan, int gamma);
QC_API int qc_decode_es_launches(const qc_plan* plan, int gamma, int iters);

/* lane-major outputs (DecodeResult / DecodedFrame layout, bp.py:87-100,
 * convolutional.py:166-177): post (n, gamma) fp32 -> post_out (gamma_out, n)
 * fp64 and/or bits_out (gamma_out, n) u8 for the first gamma_out lanes
 * (either output may be NULL). */
QC_API int qc_lane_major(int n, int gamma, int gamma_out, const float* post, double* post_out,
                  uint8_t* bits_out, void* stream);
/* same with an fp32 posterior output (half the device->host bytes) */
QC_API int qc_lane_major_f32(int n, int gamma, int gamma_out, const float* post, float* post_out,
                             uint8_t* bits_out, void* stream);
/* host-array forms (StreamDecoder.push_frame, convolutional.py:220-246): the
 * lane-major conversion into device staging (post_dev, bits_dev) followed by
 * asynchronous copies to the host arrays (page-locked for true asynchrony); and
 * an asynchronous copy of lane-major host values into x_dev followed by
 * qc_llr_from_lane_major.  Stream-ordered; the caller synchronises. */
QC_API int qc_lane_major_to_host(int n, int gamma, int gamma_out, const float* post, double* post_dev,
                                 uint8_t* bits_dev, double* post_host, uint8_t* bits_host, void* stream);
QC_API int qc_llr_from_host(int n, int gamma, int gamma_in, const double* x_host, double* x_dev, double sigma,
                            float* mu_vm, void* stream);
/* lane-major fp64 -> variable-major fp32 LLRs, lanes >= gamma_in padded with +50:
 * sigma > 0: x are received values, mu = clip((2 x)/(sigma sigma), +-50) (channel_llrs, bp.py:54-56);
 * sigma <= 0: x are LLRs, mu = clip(x, +-50) (decode_llr_batch, bp.py:231). */
QC_API int qc_llr_from_lane_major(int n, int gamma, int gamma_in, const double* x, double sigma,
                                  float* mu_vm, void* stream);

/* ---- host-buffer decode (decode_batch / decode_llr_batch, bp.py:213-274) ---
 * The reference's public decode with caller-owned HOST arrays: x (gamma, N)
 * fp64 lane-major received values (sigma > 0) or LLRs (sigma <= 0); outputs
 * bits (gamma, N) u8, post (gamma, N) fp64, ok (gamma) u8 (syndrome_ok),
 * iters_run (gamma) i64 -- DecodeResult (bp.py:87-100); bits/post/ok/iters_run
 * may each be NULL.  Chunks of `chunk` lanes rotate over `slots` CUDA streams
 * (copy-in, graph-replayed decode and copy-out overlap); page-locked host
 * arrays are DMA'd in place, pageable ones staged.  The call returns when the
 * outputs are in host memory.  A qc_host_dec is bound to the device current
 * at creation, keeps a pointer to `plan` (which must outlive it) and is not
 * thread-safe (one caller at a time). */
typedef struct qc_host_dec qc_host_dec;
QC_API int qc_host_create(const qc_plan* plan, int chunk, int slots, int iters, int early_stop,
                          qc_host_dec** out);
QC_API void qc_host_destroy(qc_host_dec* dec);
/* 1 if [p, p + bytes) is page-locked host memory (DMA'd in place), else 0 */
QC_API int qc_host_is_pinned(const void* p, size_t bytes);
/* dims: chunk, slots, iters, early_stop, device */
QC_API int qc_host_dims(const qc_host_dec* dec, int64_t* dims);
QC_API int qc_host_decode(qc_host_dec* dec, const double* x, int gamma, double sigma, uint8_t* bits,
                          double* post, uint8_t* ok, int64_t* iters_run);

/* ---- lane-recycling early-stop campaign engine (harness.py:144-204 with
 * early_stop=True): a lane whose codeword froze (bp.py:242-256) or hit the
 * iteration cap immediately starts codeword next_id; per-codeword results and
 * per-batch counters equal the reference's.  Regular (J, 24) QC grids,
 * gamma % 64 == 0.  state: qc_rc_state_bytes(gamma) bytes of device memory. */
QC_API size_t qc_rc_state_bytes(int gamma);
QC_API int qc_rc_init(int gamma, int64_t id_limit, void* state, void* stream);
/* run `ticks` flooding iterations of every busy lane; codeword id k of this rank
 * is reference batch (k / gamma_ref) * world + rank, lane lane_base + batch *
 * gamma_ref + k % gamma_ref; finished codewords add (1, bit errors, frame
 * error) to counts[batch] (n_batches x 3 int64). */
QC_API int qc_rc_ticks(const qc_plan* plan, int gamma, int gamma_ref, int world, int rank, int max_it,
                       int64_t id_limit, int64_t n_batches, uint64_t seed_lo, uint64_t seed_hi,
                       uint64_t lane_base, double sigma, int ticks, float* mu, float* msgs, uint32_t* hb,
                       void* state, int64_t* counts, void* stream);
/* copy the next codeword id (progress) to a device int64 */
QC_API int qc_rc_next_id(int gamma, const void* state, int64_t* next_id_dev_out, void* stream);

/* ---- float64 conformance build (block decoder) ---------------------------
 * The reference's own arithmetic (tanh rule with sequential forward/backward
 * products, bp.py:120-188) in float64 on the GPU, for callers relying on the
 * reference's 1e-12 tolerances.  Same layouts with double packages. */
QC_API int qc64_init(const qc_plan* plan, int gamma, const double* mu, double* msgs, void* stream);
QC_API int qc64_cnu(const qc_plan* plan, int gamma, double* msgs, const uint32_t* active, void* stream);
QC_API int qc64_vnu(const qc_plan* plan, int gamma, double* msgs, const double* mu, double* post,
                    uint32_t* hb, const uint32_t* active, void* stream);
QC_API int qc64_hard_bits(const qc_plan* plan, int gamma, const double* post, uint32_t* hb, void* stream);
QC_API int qc64_decode(const qc_plan* plan, int gamma, int iters, int early_stop, const double* mu,
                       double* msgs, double* post, uint32_t* hb, uint32_t* work, uint8_t* ok,
                       int32_t* iters_run, void* stream);
QC_API int qc64_lane_major(int n, int gamma, int gamma_out, const double* post, double* post_out,
                           uint8_t* bits_out, void* stream);
/* lane-major fp64 -> variable-major fp64 mu; sigma > 0: (2x)/(sigma sigma); clip: saturate +-50 */
QC_API int qc64_mu_from_lane_major(int n, int gamma, int gamma_in, const double* x, double sigma,
                                   int clip, double* mu, void* stream);

/* ---- channel (channel.py:61-105) ---------------------------------------- */
/* y[g, k] = 1 + sigma * ndtri(u(philox word at position start+k of lane lane0+g)),
 * mu = clip(2y/sigma^2, +-50) (bp.py:54-56).  Outputs (any may be NULL):
 *   mu_vm  (n, gamma) fp32 variable-major LLRs,
 *   y_lm   (gamma, n) fp64 lane-major received values,
 *   g_lm   (gamma, n) fp64 lane-major standard normals (lane_normals). */
QC_API int qc_channel(uint64_t seed_lo, uint64_t seed_hi, uint64_t lane0, uint64_t start, int n,
               int gamma, double sigma, float* mu_vm, double* y_lm, double* g_lm,
               void* stream);
/* Same, first lane read from device memory (*lane0_dev) so a captured CUDA
 * graph can be replayed for successive batches. */
QC_API int qc_channel_dev(uint64_t seed_lo, uint64_t seed_hi, const uint64_t* lane0_dev, uint64_t start,
                          int n, int gamma, double sigma, float* mu_vm, void* stream);
/* *lane0_dev += k */
QC_API int qc_lane_advance(uint64_t* lane0_dev, uint64_t k, void* stream);

/* ---- campaign counters (harness.py:144-154) ----------------------------- */
/* counts[b] = (frames, bit_errors, frame_errors) of lanes [b*gamma_ref, (b+1)*gamma_ref),
 * counts (gamma/gamma_ref, 3) int64, accumulated (+=). */
QC_API int qc_batch_counts(int gamma, int gamma_ref, const int32_t* lane_bits, int64_t* counts,
                    void* stream);

/* ---- LDPCCC stream decoder (convolutional.py:180-357) ------------------- */
/* Unwrapped code plan from the QC grid (LdpcccCode, convolutional.py:67-151). */
QC_API int cc_plan_create(const int64_t* shifts, int J, int L, int p, cc_plan** out);
QC_API void cc_plan_destroy(cc_plan* plan);
/* dims: lam, ms, c, cb, edge_count, sub_j, sub_l, p */
QC_API int cc_plan_dims(const cc_plan* plan, int64_t* dims);
/* One time slot of StreamDecoder._advance (convolutional.py:252-337):
 * entry of frame t, I check-layer updates, I frame updates, emission.
 *   msg   (I*E, gamma) fp32 message store,
 *   ring  (I*(ms+1), c, gamma) fp32 channel-LLR ring,
 *   mu_in (c, gamma) fp32 LLRs of frame t (NULL = zero-LLR virtual frame, flush),
 *   post_out (c, gamma) fp32 posterior of the emitted frame t-I(ms+1)+1 (may be NULL),
 *   lane_cnt (3, gamma) i32 (may be NULL): row 0 = bit count of the frame emitted
 *   by the previous slot (folded by the next slot's entry kernel), row 1 += bit
 *   errors, row 2 += frame errors of every emitted frame (harness.py:228-232);
 *   call cc_fold after the last slot of a segment.
 * t_dev: if non-NULL the slot index is *t_dev + t (device-resident slot
 * counter, so a CUDA graph of K slots can be replayed; see cc_advance). */
QC_API int cc_slot(const cc_plan* plan, int I, int gamma, int64_t t, const int64_t* t_dev, float* msg,
            float* ring, const float* mu_in, float* post_out, int32_t* lane_cnt, void* stream);
/* Part of slot t: parts bit 0 = entry of frame t, bit 1 = check phase, bit 2 =
 * variable phase, of processors [ip0, ip0 + nip) only (0-based; processor I-1
 * emits).  Within a slot the processors' (check, variable) pairs and the entry
 * touch disjoint edges and ring slots, so the emitting processor can run
 * first and the rest after it -- StreamDecoder.push_frame returns the emitted
 * frame while the other I-1 processors and the next frame's copy-in proceed.
 * cc_slot = cc_slot_part(..., 0, I, 7, ...). */
QC_API int cc_slot_part(const cc_plan* plan, int I, int gamma, int64_t t, const int64_t* t_dev, float* msg,
                        float* ring, const float* mu_in, float* post_out, int32_t* lane_cnt, int ip0, int nip,
                        int parts, void* stream);
/* Look-ahead slot for device-resident campaigns (harness.py:226-232 with every
 * frame's LLRs known up front): the check and variable phases of slot t, where
 * the check phase folds the previous emission's count (the entry kernel's job
 * in cc_slot) and, when enter_next != 0, the emitting processor's variable
 * threads enter frame t + 1 from mu_next (NULL = zero-LLR virtual frame) right
 * after emitting frame t + 1 - I(ms+1), which used the same ring slot and edge
 * slots.  Two launches per slot instead of three; frame 0 is entered with
 * cc_slot_part(parts = 1).  Results equal cc_slot bit for bit. */
QC_API int cc_slot_ahead(const cc_plan* plan, int I, int gamma, int64_t t, const int64_t* t_dev, float* msg,
                         float* ring, const float* mu_next, int enter_next, float* post_out, int32_t* lane_cnt,
                         void* stream);
/* fold the last emitted frame's count into lane_cnt rows 1-2 (end of segment) */
QC_API int cc_fold(int32_t* lane_cnt, int gamma, void* stream);
/* *t_dev += k (ends a graph of k slots). */
QC_API int cc_advance(int64_t* t_dev, int64_t k, void* stream);
/* Channel for stream segments: frame t of lanes lane0.. at positions t*c
 * (harness.py:226-227), LLRs straight into mu (c, gamma); t_dev as in cc_slot. */
QC_API int cc_channel(const cc_plan* plan, uint64_t seed_lo, uint64_t seed_hi, uint64_t lane0,
                      const uint64_t* lane0_dev, int64_t t, const int64_t* t_dev, int gamma,
                      double sigma, float* mu, void* stream);
/* Frames t .. t + nframes - 1 in one launch (contiguous positions t*c ..), into
 * mu (nframes, c, gamma): amortises the channel over several slots. */
QC_API int cc_channel_frames(const cc_plan* plan, uint64_t seed_lo, uint64_t seed_hi, uint64_t lane0,
                             const uint64_t* lane0_dev, int64_t t, int nframes, int gamma, double sigma,
                             float* mu, void* stream);

#ifdef __cplusplus
}
#endif
#endif
