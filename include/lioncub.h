/*
 * lioncub.h — C ABI of the B200-native Lion Cub distributed optimizer step.
 *
 * Everything is plain pointers, sizes and scalars (no torch types).  Device
 * pointers point into CUDA global memory of the calling thread's current
 * device; `stream` is a cudaStream_t passed as void*.  Every entry point
 * returns 0 (LC_OK) or a negative LC_E_* code; lc_last_error() gives the
 * thread-local message.  Kernels are enqueued asynchronously on `stream`.
 *
 * The reference (lioncomm, pure numpy, /root/reference/pkg/src/lioncomm) has
 * no native code; each entry point below names the reference function whose
 * per-layer numpy computation it replaces (file:line).  The Python host side
 * (paper_2411_16462_b200/optimizer.py, collectives.py) keeps the reference's
 * API and calls these through ctypes; INTEGRATION.md shows the binding.
 */
#ifndef LIONCUB_H_
#define LIONCUB_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define LIONCUB_ABI_VERSION 4

enum {
  LC_OK = 0,
  LC_E_CONFIG = -1,     /* -> ConfigError      (errors.py:8)            */
  LC_E_CAPACITY = -2,   /* -> CapacityError    (errors.py:12-16)        */
  LC_E_COLLECTIVE = -3, /* -> CollectiveError  (errors.py:35-52)        */
  LC_E_CUDA = -4,       /* CUDA runtime failure                          */
  LC_E_ARG = -5         /* bad pointer / size / alignment                */
};

/* Device flag bits written by the kernels (checked by the host shim). */
enum {
  LC_FLAG_ZERO_SIGN = 1u << 0, /* exact zero on a path that cannot carry it
                                  (collectives.py:264-267, :202-203)        */
  LC_FLAG_NAN = 1u << 1,       /* NaN in c (reference: PackRangeError)      */
  LC_FLAG_TIE_TERNARY = 1u << 2, /* tied 1-bit vote in exact-ternary mode
                                    (collectives.py:290-293)               */
  LC_FLAG_RANGE = 1u << 3,     /* |q| > q_max / non-binary value
                                  (collectives.py:202-208)                  */
  LC_FLAG_BARRIER_TIMEOUT = 1u << 4 /* a peer never reached lc_barrier     */
};

/* Encodings produced by the fused interpolate pass (lc_encode). */
enum {
  LC_ENC_SIGN1 = 0,       /* 1-bit sign words (compressed1bit)            */
  LC_ENC_SIGN_FIELDS = 1, /* (s+1)>>1 in F-bit fields (sum-of-signs)      */
  LC_ENC_QUANT_FIELDS = 2,/* q+q_max in F-bit fields (L1 p-bit)           */
  LC_ENC_F64 = 3,         /* c as float64 (full-precision ps arm)         */
  LC_ENC_REPLICATE = 0x100 /* OR with LC_ENC_SIGN1: every dst gets all words
                              (allgather of the payload; L >= eoff+n)      */
};

typedef struct lc_hyper {
  double beta1, one_minus_beta1; /* 1-b1 computed on the host in f64 */
  double beta2, one_minus_beta2;
  double lr;                     /* eta_t = LionHyper.lr_at(t)        */
  double weight_decay;
} lc_hyper;

/* In-kernel cross-GPU barrier (peer-memory exchange).  A kernel given a
 * sync with wait_epoch != 0 first waits (one thread per peer polling with
 * ld.acquire.sys, timeout -> LC_FLAG_BARRIER_TIMEOUT in *err) until every
 * peer published wait_epoch into my_flags; a kernel given arrive_epoch != 0
 * publishes it into every peer's flag slot `rank` after its last CTA
 * finished (per-CTA fence + atomic counter, st.release.sys).  This replaces
 * a separate barrier launch between K1 -> vote -> K5.  NULL = no sync. */
#define LC_SYNC_COUNTER_WORDS 8
typedef struct lc_sync {
  void* peer_flags[32]; /* rank j's uint64[P] flag array, mapped here     */
  uint64_t* my_flags;   /* this rank's flag array                          */
  uint32_t* counter;    /* LC_SYNC_COUNTER_WORDS zeroed device words per
                           arrive site: [0] arrivals (lc_vote_apply: vote
                           units done), [1..4] lc_vote_apply's work
                           counters (update items, retired CTAs, vote
                           units claimed, CTA tickets); every kernel
                           leaves them zero                                */
  uint32_t* err;        /* 2 device words: [0] LC_FLAG_* bits, [1] bitmask
                           of the ranks a wait timed out on.  A kernel whose
                           wait times out writes nothing (theta, m and the
                           peers' buffers keep their values) and its arrival
                           publishes no epoch, so every live rank fails.   */
  uint64_t wait_epoch;
  uint64_t arrive_epoch;
  int32_t P, rank;
  double timeout_s;
  uint64_t* verdict;    /* nullable: a pinned host word.  lc_vote_apply and
                           lc_vote_update store (epoch << 8) | status into it
                           as soon as every wait of the step has resolved --
                           epoch = arrive_epoch (wait_epoch if that is 0),
                           status = the LC_FLAG_* bits of *flags (the NaN
                           flag of K1 ...) | LC_FLAG_BARRIER_TIMEOUT -- so
                           the host can check the step (lc_wait_verdict)
                           while the theta update is still running         */
} lc_sync;

/* Spin (GIL-free, from ctypes) until *word carries an epoch >= epoch; its
 * status byte goes to *status.  LC_E_COLLECTIVE if timeout_s passes first
 * (the kernels' own bounded waits normally answer long before). */
int lc_wait_verdict(const uint64_t* word, uint64_t epoch, double timeout_s, uint32_t* status);

/* Quantizer variant flags (QuantSpec, quant.py:28-55). */
enum {
  LC_Q_STOCHASTIC = 1u << 0, /* rounding="stochastic": floor(v) + (u < frac),
                                u from the counter-based stream lc::uniform01(seed, e)
                                (reference: PCG64 draws, quant.py:107-116)   */
  LC_Q_NO_ZERO = 1u << 1     /* no_zero: q == 0 and c != 0 -> sign(c) (:171-173) */
};

/* Per-layer segment table of a flat buffer (layers in sorted-name order).
 * The quantizer (quant.py:127-173) is q = clip(round(scale[s] * y), +-qmax)
 * with y = c, or y = sign(c) log1p(|c| / log_scale[s]) when log_scale is
 * given and log_scale[s] > 0 (log_transform, quant.py:143-146). */
typedef struct lc_segments {
  const int64_t* start; /* device, nseg+1 offsets (elements)               */
  const double* scale;  /* device, nseg scales: qmax/(2 M_p), or qmax/M_inf
                           for norm_p = inf; NULL when not quantizing      */
  int32_t nseg;
  int32_t qmax;
  const double* log_scale; /* device, nseg M1(c) for log_transform, or NULL */
  uint32_t qflags;         /* LC_Q_* bits                                   */
  uint32_t reserved;
  uint64_t seed;           /* stochastic-rounding stream of this rank/step  */
} lc_segments;

int lc_abi_version(void);
const char* lc_last_error(void);
int lc_device_sm_count(int device);
/* Share the GPU among `divisor` ranks that launch concurrently from separate
 * host threads onto one device (simulated ranks of the peer-memory exchange,
 * transport.LocalTransport(fused=True)): every grid this host thread sizes
 * from the SM count uses SMs/divisor, so all ranks' barrier-waiting kernels
 * are co-resident.  Thread-local; 1 (the default) = the whole GPU. */
int lc_set_grid_divisor(int divisor);

/* Maximum entries of a destination / peer table (blocks of a packed vector). */
#define LC_MAX_BLOCKS 64

/* ---- K1: fused Lion interpolate + sign/quantize + pack + momentum EMA ----
 * Replaces optimizer.py:199-201 (c, mask), :205 (m'), quant.py:198-204
 * (apply_sign), quant.py:255-281 (pack width 1 / F-bit fields),
 * quant.py:161-168 (finite-p quantize given the per-layer scale), and the
 * offsetting of collectives.py:201-210.  Computes c and m' in float64 from
 * fp32 g,m (no FMA contraction) and writes m' (fp32) in place.
 *   fill: +1 / -1 = alternating zero fill (quant.py:76-78), 0 = ternary.
 *   field_bits: 1 for SIGN1, F in {1,2,4,8,16,32} for *_FIELDS, 64 for F64.
 *   dst[j], j < nblocks: where block j (elements [j*L, (j+1)*L)) of the
 *     packed vector goes -- uint32 words (L*F/32 per block) or doubles.
 *     A local send buffer ([P][L*F/32] for an NCCL exchange) or, for the
 *     NVLink path, the owner GPU's receive slot (peer pointer), so the
 *     all-to-all happens inside the kernel.  L is a multiple of 1024.
 *   eoff: index of g[0]/m[0] in the full vector (multiple of 1024), so a
 *     chunk of the vector can be encoded as soon as it arrives.
 *   g, m must be 16-byte aligned. mask may be NULL (uint8 per element). */
int lc_encode(const float* g, float* m, const uint8_t* mask, int64_t n,
              const lc_hyper* h, int fill, int enc, int field_bits,
              const lc_segments* segs, void* const* dst, int32_t nblocks,
              int64_t L, int64_t eoff, uint32_t* flags, const lc_sync* sync,
              void* stream);

/* Output tables of the owner-side vote kernels: voted/nz/tie_bits are host
 * arrays of `nout` word pointers; the owner's block is written to every one
 * (nout = 1: local gather buffer before an NCCL allgather; nout = P: every
 * rank's gather buffer over NVLink, i.e. the allgather inside the kernel;
 * nout = -1: each table holds ONE NVLS multicast address and a single
 * multimem.st reaches every rank's gather buffer through the NVSwitch).
 * nz / tie_bits may be NULL.  nz marks non-zero aggregates (exact-ternary),
 * tie_bits marks aggregates that are exactly 0 (VoteResult.ties). */

/* ---- K4: owner-side 1-bit majority vote over P packed chunks ----
 * Replaces collectives.py:288-293 (stack+sum, local ties, apply_sign).
 * recv: [P][cw] words (cw % 4 == 0); n_valid: real elements in the chunk.
 * sum_mode 0 = compressed1bit (exact-ternary tie -> LC_FLAG_TIE_TERNARY);
 * sum_mode 1 = sum-of-signs (the tally is the exact p-bit sum 2k-P,
 * collectives.py:241-248; a zero sum is a zero update in exact-ternary). */
int lc_vote_bits(const uint32_t* recv, int32_t P, int64_t cw, int64_t n_valid,
                 int fill, int sum_mode, void* const* voted, void* const* nz,
                 void* const* tie_bits, int32_t nout, uint32_t* flags,
                 const lc_sync* sync, void* stream);

/* ---- K4+K5 fused (peer-memory path, 1-bit words): vote this owner's block
 * (as lc_vote_bits, voted/nz pushed through the nout table), publish
 * sync->arrive_epoch, then update theta (as lc_apply_update from the local
 * gather buffer `full`/`nz_full`), each warp waiting only for the owner of
 * the block it reads (peer flag >= arrive_epoch).  sync->wait_epoch: all
 * ranks' encode finished.  P <= 32. */
int lc_vote_apply(const uint32_t* recv, int32_t P, int64_t cw, int64_t n_valid,
                  int fill, int sum_mode, void* const* voted, void* const* nz,
                  int32_t nout, uint32_t* flags, const lc_sync* sync, float* theta,
                  int64_t n, const uint32_t* full, const uint32_t* nz_full, double lr,
                  double weight_decay, void* stream);

/* ---- The momentum sync fused into the step (SyncPolicy(layers="all")
 * firing at this step; maybe_sync_momentum, optimizer.py:244-258, with
 * allreduce_mean_f32, collectives.py:319-344) ----
 * lc_encode_sync (sync required, sync->P == nblocks): the 1-bit encode (as
 *   lc_encode, LC_ENC_SIGN1, eoff 0) that
 *   stores m' of block j into mstage[j] -- owner j's staging row for this
 *   rank (L floats, 16-byte aligned) -- instead of the local m.
 * lc_vote_apply_sync: lc_vote_apply plus the owner mean: this owner's P
 *   staged rows (mean_stage + r*mean_L, r in rank order) summed in float64,
 *   divided once, rounded once to fp32 and stored into every rank's momentum
 *   block (mean_out[k], k < P); mean_cnt valid elements; mean_work: a device
 *   word the call zeroes (CTAs take 8192-element chunks from it).  The mean
 *   needs only sync->wait_epoch (every rank's lc_encode_sync finished).  The
 *   caller orders the next step after every owner's mean (a barrier).
 *   side_stream: run the mean as its own kernel on that stream, concurrently
 *   with the vote/update grid (capped to leave it SMs), joined back into
 *   `stream`; NULL: every vote/update CTA joins the mean after its share. */
/* Cap the grid of this host thread's next lc_vote_apply launches at
 * ctas_per_sm CTAs per SM (0 = occupancy-sized), leaving SMs to a kernel
 * the caller runs concurrently on another stream (the selective momentum
 * sync's pull, fused into the step).  Thread-local. */
int lc_set_vote_cap(int32_t ctas_per_sm);
/* The owner mean of the fused sync on its own (as lc_vote_apply_sync's side
 * kernel; stand-alone for tuning and the NVLink microbenchmark): wait
 * (nullable) -> wait_epoch only; ctas_per_sm > 0 caps the grid. */
int lc_sync_mean(const lc_sync* wait, const float* stage, void* const* out, int32_t P, int64_t L,
                 int64_t cnt, uint32_t* work, int32_t ctas_per_sm, void* stream);
int lc_encode_sync(const float* g, float* m, const uint8_t* mask, int64_t n,
                   const lc_hyper* h, int fill, void* const* dst, int32_t nblocks, int64_t L,
                   uint32_t* flags, const lc_sync* sync, void* const* mstage, void* stream);
int lc_vote_apply_sync(const uint32_t* recv, int32_t P, int64_t cw, int64_t n_valid,
                       int fill, int sum_mode, void* const* voted, void* const* nz,
                       int32_t nout, uint32_t* flags, const lc_sync* sync, float* theta,
                       int64_t n, const uint32_t* full, const uint32_t* nz_full, double lr,
                       double weight_decay, const float* mean_stage, void* const* mean_out,
                       int64_t mean_L, int64_t mean_cnt, uint32_t* mean_work,
                       void* side_stream, void* stream);

/* ---- K5v: vote + theta update over allgathered sign words ----
 * rows: P rows (stride row_stride >= ceil(n/32) words) of every rank's
 * 1-bit sign words for the whole vector (lc_encode with LC_ENC_REPLICATE
 * stores row `rank` into every rank's buffer).  Each word is voted from the
 * P rows (the owner vote of lc_vote_bits: majority / sum-of-signs, fill,
 * exact-ternary flags) and theta updated in the same pass (lc_apply_update).
 * sync->wait_epoch: every rank's encode finished.  Replaces collectives.py
 * :287-299 + optimizer.py:204 on the allgather exchange. */
int lc_vote_update(const uint32_t* rows, int64_t row_stride, int32_t P, float* theta,
                   int64_t n, int fill, int sum_mode, double lr, double weight_decay,
                   uint32_t* flags, const lc_sync* sync, void* stream);

/* ---- K6: owner-side p-bit sums -> signed aggregate -> 1-bit vote ----
 * Replaces collectives.py:241-249 (de-offset, ties) + :313-316
 * (majority_sign).  sums: `rows` rows (stride row_stride words) of F-bit
 * fields whose word-wise sum is the field sum over ranks (rows = 1 after an
 * NCCL reduce-scatter, rows = P when peers wrote over NVLink).
 * offset: q_max (0 with binary=1 for sum-of-signs, signed = 2k-P).
 * values (nullable): signed aggregate as int64 (VoteResult.values). */
int lc_fields_vote(const uint32_t* sums, int32_t rows, int64_t row_stride,
                   int64_t n, int32_t field_bits, int32_t P, int32_t offset,
                   int32_t binary, int fill, void* const* voted, void* const* nz,
                   void* const* tie_bits, int32_t nout, int64_t* values,
                   const lc_sync* sync, void* stream);

/* ---- full-precision arm: P float64 rows (row stride `stride`) -> sum of
 * the first `len` elements in the reference's rank order (flat,
 * collectives.py:153-158, or binomial tree :96-109) -> sign words.
 * values (nullable) receives the f64 sum.  nout <= 32. */
int lc_f64_sum_vote(const double* recv, int32_t P, int64_t len, int64_t stride,
                    int tree, int fill, void* const* voted, void* const* nz,
                    void* const* tie_bits, int32_t nout, double* values,
                    const lc_sync* sync, void* stream);

/* ---- K5: theta' = theta - eta*(s + wd*theta)  (optimizer.py:204) ----
 * s = +1/-1 from the voted sign bits; 0 where nz_bits has a 0 bit.
 * sign_bits / nz_bits (nullable) are tables of nsrc word arrays indexed by
 * the GLOBAL word index; word w is read from table entry w / wpb -- the
 * owner of that block.  nsrc = 1: local gather buffer; nsrc = P: each
 * owner's vote output over NVLink (the allgather pulled inside K5).
 * woff: global word index of theta[0] / 32 (chunked updates). */
int lc_apply_update(float* theta, int64_t n, void* const* sign_bits,
                    void* const* nz_bits, int32_t nsrc, int64_t wpb, int64_t woff,
                    double lr, double weight_decay, const lc_sync* sync,
                    void* stream);

/* ---- one-pass step for P == 1 (no exchange: the vote of one rank is its
 * own aggregate): reads theta,m,g, writes theta',m' (20 B/param).
 * mode: LC_LOCAL_BINARY  sign(c) with the fill BEFORE aggregation
 *                        (compressed1bit, direct bits=1; a zero in
 *                        exact-ternary mode sets LC_FLAG_ZERO_SIGN),
 *       LC_LOCAL_PS      aggregate = c (ps, spec=None), ties = #(c==0),
 *       LC_LOCAL_QUANT   aggregate = L1-quantized c (needs segs->scale).
 * Optional metric outputs (nullable): sign_bits/nz_bits = applied sign,
 * tie_bits = aggregate exactly zero. */
enum { LC_LOCAL_BINARY = 0, LC_LOCAL_PS = 1, LC_LOCAL_QUANT = 2 };
int lc_fused_local_step(float* theta, float* m, const float* g,
                        const uint8_t* mask, int64_t n, const lc_hyper* h,
                        int fill, int mode, const lc_segments* segs,
                        uint32_t* sign_bits, uint32_t* nz_bits,
                        uint32_t* tie_bits, uint32_t* flags, void* stream);

/* ---- K7: momentum mean (collectives.py:336-340): f64 rank-ordered sum of P
 * fp32 rows (row stride in elements), /P, one rounding to fp32. */
int lc_mean_f32(const float* recv, int32_t P, int64_t len, int64_t stride,
                float* out, void* stream);

/* ---- L1 norm per segment, numpy-exact (quant.py:81-104, p=1):
 * M1 = max|c| * (pairwise_sum(|c|/max) / n) with numpy's pairwise
 * summation order reproduced exactly; c recomputed from g,m,mask.
 * Writes per-segment norms and scale = qmax/(2 M1) (0 if M1 == 0),
 * quant.py:161.  The plan holds the summation-tree schedule (device). */
typedef struct lc_l1_plan_s* lc_l1_plan_t;
int lc_l1_plan_create(lc_l1_plan_t* plan, const int64_t* seg_start_host,
                      int32_t nseg);
int lc_l1_plan_destroy(lc_l1_plan_t plan);
int lc_l1_scales(lc_l1_plan_t plan, const float* g, const float* m,
                 const uint8_t* mask, const lc_hyper* h, int32_t qmax,
                 double* norms, double* scales, void* stream);
/* ---- per-segment mean p-norm of every order (quant.py:81-104) and the
 * quantizer scale, for y = c or the log-mapped c (log_scale != NULL):
 *   p = 1    exact (the lc_l1_scales schedule);
 *   p = 2, 0.5  exact: (a/max)**2 = square, **0.5 = sqrt, as numpy does;
 *   other finite p  max * mean(pow(a/max, p))**(1/p) in numpy's pairwise
 *            order, CUDA pow (<= 2 ulp; numpy's own pow is not glibc's);
 *   p = 0    exp(sum(log a) / #nonzero) (tree order, CUDA log/exp);
 *   p = inf  max|y|, scale = qmax / M.
 * norms/scales: nseg doubles each. */
typedef struct lc_norm_spec {
  double p;                /* 0, finite > 0, or +inf                        */
  int32_t qmax;
  int32_t reserved;
  const double* log_scale; /* device, nseg M1(c) (from lc_l1_scales), or NULL */
} lc_norm_spec;
int lc_norm_scales(lc_l1_plan_t plan, const float* g, const float* m,
                   const uint8_t* mask, const lc_hyper* h, const lc_norm_spec* spec,
                   double* norms, double* scales, void* stream);
/* Self-check of the reciprocal-based correctly rounded division the norm
 * kernel uses for |c|/max (counts bit mismatches vs IEEE division over
 * pairs with |a| clamped to b). */
int lc_debug_div_check(const double* a, const double* b, int64_t n,
                       uint64_t* mismatches, void* stream);

/* ---- standalone quantizer operators (quant.py; csrc/quant.cu) ----
 * lc_quantize_values: q = quantize(x) elementwise (quant.py:151-173) with the
 *   segment table of lc_norm_scales (qmax, scale, log_scale, qflags, seed);
 *   the stochastic stream position of x[e] is e.
 * lc_dequantize: y = q * mult (mult = norm/qmax for p = inf, else
 *   2 norm/qmax, computed by the caller as numpy does); log != 0 undoes the
 *   log map: sign(y) * log_scale * expm1(|y|) (quant.py:176-195).
 * lc_apply_sign_values: apply_sign (quant.py:198-204) of a float32
 *   (is_f64 = 0) or float64 vector: +-1, zeros (and -0.0) -> fill in
 *   {+1, -1, 0}; NaN -> 0.
 * lc_f64_to_f32_exact: float64 -> float32, LC_FLAG_RANGE when a value is
 *   not exactly representable (the CUDA operators compute from fp32). */
int lc_quantize_values(const float* x, int64_t n, const lc_segments* segs,
                       int64_t* q, void* stream);
int lc_dequantize(const int64_t* q, int64_t n, double mult, double log_scale,
                  int32_t log, double* out, void* stream);
int lc_apply_sign_values(const void* x, int32_t is_f64, int64_t n, int fill,
                         int8_t* out, void* stream);
int lc_f64_to_f32_exact(const double* x, int64_t n, float* out, uint32_t* flags,
                        void* stream);

/* ---- metrics / operator helpers ---- */
/* Momentum divergence (optimizer.py:261-276): per segment, the max over its
 * elements of the population std across P fp32 rows (row r at rows + r*stride),
 * numpy's rank-ordered float64 mean / sum of squares; bit-exact. */
int lc_std_max_segmented(const float* rows, int32_t P, int64_t n, int64_t stride,
                         const int64_t* seg_start, int32_t nseg, double* out_max,
                         void* stream);
/* Vote sign vs the sign of the full-precision aggregate (runner.py:171-177):
 * counts[0] = #(vote == sign(ref) and vote != 0), counts[1] = #(vote ==
 * -sign(ref), both nonzero); ref = allreduce_mean_f32(c_local). */
int lc_sign_agreement(const int8_t* vote, const float* ref, int64_t n, int64_t* counts,
                      void* stream);
/* c as float64 (metrics_out["c_local"], optimizer.py:209). */
int lc_compute_c(const float* g, const float* m, const uint8_t* mask,
                 int64_t n, const lc_hyper* h, double* c, void* stream);
/* Per-segment popcount of bit words (ties per layer, optimizer.py:207). */
int lc_count_bits_segmented(const uint32_t* bits, const int64_t* seg_start,
                            int32_t nseg, int64_t* counts, void* stream);
/* bits -> int8 +-1 (0 where nz bit is 0): vote_sign (optimizer.py:208). */
int lc_bits_to_sign(const uint32_t* sign_bits, const uint32_t* nz_bits,
                    int64_t n, int8_t* out, void* stream);
/* int64 values -> F-bit fields of v+offset (binary: (v+1)>>1), range check
 * into flags (collectives.py:201-210, quant.py:255-281). */
int lc_pack_i64_fields(const int64_t* v, int64_t n, int32_t field_bits,
                       int32_t offset, int32_t binary, uint32_t* out,
                       uint32_t* flags, void* stream);
/* F-bit fields of sums -> signed int64 aggregate (collectives.py:241-247). */
int lc_fields_decode(const uint32_t* sums, int64_t n, int32_t field_bits,
                     int32_t P, int32_t offset, int32_t binary, int64_t* out,
                     void* stream);
/* Exact-ternary pre-flight of the binary paths (collectives.py:262-267,
 * :202-203): sign(c) of c = beta1*m + (1-beta1)*g (masked) for every element,
 * LC_FLAG_ZERO_SIGN in *flags if any is zero, and -- when out is not NULL --
 * the sign words (bit = c > 0) for the owner tie check of the 1-bit vote.
 * Reads g, m only (8 B/param; m is not written). */
int lc_sign_check(const float* g, const float* m, const uint8_t* mask, int64_t n,
                  const lc_hyper* h, uint32_t* out, uint32_t* flags, void* stream);
/* sign of a float64/float32 vector with fill -> 1-bit words (K1 without
 * the Lion interpolation; compressed_allreduce_1bit on raw c). */
int lc_sign_pack_f64(const double* c, int64_t n, int fill, uint32_t* out,
                     uint32_t* flags, void* stream);
/* Sum of P uint32 rows into out (the in-process transport's reduce). */
int lc_sum_u32_rows(const uint32_t* const* rows, int32_t P, int64_t count,
                    uint32_t* out, void* stream);

/* ---- NCCL transport (one communicator per GPU rank) ----
 * The reference's plugin boundary is Transport.send/recv (transport.py:32-45);
 * on B200 the collective boundary is an NCCL communicator over NVLink. */
typedef struct lc_comm_s* lc_comm_t;
int lc_nccl_version(void);
int lc_nccl_unique_id(uint8_t out[128]);
int lc_comm_init_rank(lc_comm_t* comm, const uint8_t id[128], int32_t nranks,
                      int32_t rank);
int lc_comm_init_all(lc_comm_t* comms, int32_t ndev, const int32_t* devices);
/* `count` communicators initialised together (ncclGroupStart/End around the
 * ncclCommInitRank calls): ids[128*i], nranks[i], ranks[i].  Used for the
 * per-direction pair communicators of the frame transport. */
int lc_comm_init_group(lc_comm_t* comms, const uint8_t* ids, const int32_t* nranks,
                       const int32_t* ranks, int32_t count);
/* Point-to-point bytes (ncclSend / ncclRecv) on `stream`: the frames of
 * Transport.send/recv (transport.py:32-45) over NVLink. */
/* Establish the NCCL p2p connections of 2-rank pair communicators in one
 * group (a 1-byte send / receive on each, on its own device and stream):
 * the first p2p call on a communicator connects it and blocks until the
 * peer joins, so connecting lazily from threads that each send first would
 * deadlock. */
int lc_pair_connect(const lc_comm_t* comms, const int32_t* is_send, void* const* scratch,
                    void* const* streams, int32_t count);
int lc_send_bytes(lc_comm_t comm, const void* buf, int64_t bytes, int32_t peer, void* stream);
int lc_recv_bytes(lc_comm_t comm, void* buf, int64_t bytes, int32_t peer, void* stream);
int lc_comm_destroy(lc_comm_t comm);
int lc_comm_abort(lc_comm_t comm);
/* LC_OK, or LC_E_COLLECTIVE if the communicator hit an asynchronous error. */
int lc_comm_check(lc_comm_t comm);
/* Equal-block all-to-all: block j of send goes to rank j, block i of recv
 * comes from rank i (collectives.py:276-286 stage 1). */
int lc_alltoall(lc_comm_t comm, const void* send, void* recv,
                int64_t bytes_per_peer, void* stream);
/* Variable all-to-all (host byte counts/displacements, P entries each). */
int lc_alltoallv(lc_comm_t comm, const void* send, const int64_t* send_bytes,
                 const int64_t* send_displ, void* recv,
                 const int64_t* recv_bytes, const int64_t* recv_displ,
                 void* stream);
/* AllGather; in place when send == recv + rank*bytes (collectives.py:295-306). */
int lc_allgather(lc_comm_t comm, const void* send, void* recv, int64_t bytes,
                 void* stream);
/* ReduceScatter(sum) on uint32 words of packed fields: carry-free because
 * the capacity check bounds every field sum (collectives.py:196-199,226-231). */
int lc_reduce_scatter_u32(lc_comm_t comm, const uint32_t* send, uint32_t* recv,
                          int64_t count_per_rank, void* stream);
int lc_allreduce_max_u32(lc_comm_t comm, const uint32_t* send, uint32_t* recv,
                         int64_t count, void* stream);
int lc_allreduce_sum_i64(lc_comm_t comm, const int64_t* send, int64_t* recv,
                         int64_t count, void* stream);

/* ---- NVLink peer memory (symmetric buffers) ----
 * lc_sym_alloc: cudaMalloc'ed, zeroed buffer + its 64-byte IPC handle;
 * lc_sym_open maps a peer process's handle (lc_sym_close unmaps).  With one
 * thread per GPU, lc_enable_peer_access makes raw peer pointers usable. */
int lc_sym_alloc(int64_t bytes, void** ptr, uint8_t handle[64]);
int lc_sym_free(void* ptr);
int lc_sym_open(const uint8_t handle[64], void** ptr);
int lc_sym_close(void* ptr);
int lc_enable_peer_access(int32_t device, int32_t peer);
/* Stream-ordered cross-GPU barrier: publish `epoch` into slot `rank` of every
 * peer's flag array (peer_flags[j] = rank j's uint64[P] array), then wait
 * until all P slots of my_flags reach it.  After timeout_s instead of hanging
 * it sets LC_FLAG_BARRIER_TIMEOUT in err[0] and bit j of err[1] for every
 * rank j that never arrived (-> CollectiveError naming it). */
int lc_barrier(void* const* peer_flags, int32_t P, int32_t rank, uint64_t* my_flags,
               uint64_t epoch, double timeout_s, uint32_t* err, void* stream);
/* Momentum sync over peer memory (collectives.py:319-344): push block j of a
 * fp32 vector (blocks of s) to dst[j]; the owner then averages its P rows in
 * float64 rank order and stores the fp32 mean to every out[k] (nout = -1:
 * out[0] is an NVLS multicast address, one store reaches every rank). */
int lc_push_blocks_f32(const float* src, int64_t len, int64_t s, void* const* dst,
                       int32_t P, void* stream);
int lc_mean_bcast_f32(const float* recv, int32_t P, int64_t cnt, int64_t s,
                      void* const* out, int32_t nout, void* stream);
/* Same mean without staging: the owner loads elements [off, off+cnt) of
 * every rank's momentum directly (src[j] = rank j's buffer, peer pointers)
 * and stores the fp32 mean to out (nout = -1: NVLS multicast base; else
 * nout per-rank base pointers).  Ranks' buffers must be final (barrier).
 * err (nullable): the barrier's error words -- after a timeout nothing is
 * averaged or stored. */
int lc_mean_pull_f32(void* const* src, int32_t P, int64_t off, int64_t cnt,
                     void* const* out, int32_t nout, const uint32_t* err, void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* LIONCUB_H_ */
