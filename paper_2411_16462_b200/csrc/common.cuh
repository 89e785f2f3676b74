// Shared helpers for the Lion Cub sm_100a kernels.
#pragma once

#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <string>
#include <utility>

#include "lioncub.h"

namespace lc {

constexpr unsigned kFull = 0xffffffffu;

// Thread-local error message behind lc_last_error().
std::string& err_msg();
int set_err(int code, const char* fmt, ...);

#define LC_CUDA_TRY(expr)                                                    \
  do {                                                                       \
    cudaError_t e_ = (expr);                                                 \
    if (e_ != cudaSuccess)                                                   \
      return ::lc::set_err(LC_E_CUDA, "%s: %s (%s:%d)", #expr,               \
                           cudaGetErrorString(e_), __FILE__, __LINE__);      \
  } while (0)

#define LC_LAUNCH_CHECK() LC_CUDA_TRY(cudaPeekAtLastError())

// SMs of the current device (cached per device).
int sm_count();

// Resident CTAs per SM of `kernel` at `block` threads (occupancy query),
// cached per (device, kernel) -- the query is not free on the launch path.
// Keyed by the kernel's address: template instances share a type but not
// their register counts.  Thread-safe (one host thread per GPU may launch).
int resident_ctas_of(const void* kernel, int block);

template <typename K>
int resident_ctas(K kernel, int block) {
  return resident_ctas_of(reinterpret_cast<const void*>(kernel), block);
}

// Grid size for a grid-stride streaming kernel: enough resident CTAs to fill
// every SM (occupancy-derived), never more than the work needs.
template <typename K>
int stream_grid(K kernel, int block, int64_t work_items, int items_per_cta) {
  int per_sm = resident_ctas(kernel, block);
  int64_t need = (work_items + items_per_cta - 1) / items_per_cta;
  int64_t cap = (int64_t)sm_count() * per_sm;
  int64_t g = need < cap ? need : cap;
  return g < 1 ? 1 : (int)g;
}

struct Hyp {
  double b1, omb1, b2, omb2;
};

// c = beta1*m + (1-beta1)*g in float64, each product and the sum rounded
// separately exactly like numpy (optimizer.py:199); no FMA contraction.
__device__ __forceinline__ double lion_c(float m, float g, const Hyp& h) {
  return __dadd_rn(__dmul_rn(h.b1, (double)m), __dmul_rn(h.omb1, (double)g));
}

// m' = beta2*m + (1-beta2)*g (optimizer.py:205), rounded once to fp32.
__device__ __forceinline__ float lion_m(float m, float g, const Hyp& h) {
  return __double2float_rn(
      __dadd_rn(__dmul_rn(h.b2, (double)m), __dmul_rn(h.omb2, (double)g)));
}

// theta' = theta - eta*(s + wd*theta) (optimizer.py:204), float64 then fp32.
__device__ __forceinline__ float lion_theta(float th, double s, double lr,
                                            double wd) {
  double t = (double)th;
  return __double2float_rn(
      __dsub_rn(t, __dmul_rn(lr, __dadd_rn(s, __dmul_rn(wd, t)))));
}

// Stochastic-rounding stream: element e of a rank's flat buffer draws
// u = x * 2^-32 in [0, 1), x = lowbias32(lo32(e) * 0x9E3779B9 + lo32(seed)
// ^ hi32(e) * 0x85EBCA6B ^ hi32(seed)) -- a counter-based generator (no
// per-thread state; any element range can be drawn independently) in 32-bit
// integer ops only: the splitmix64 stream it replaces spent ~35 issue slots
// per element on 64-bit multiplies and left the stochastic step issue-bound.
// For a fixed seed and hi32(e) the map lo32(e) -> x is a bijection, so no
// two of 2^32 consecutive elements share a draw; the 32-bit resolution
// biases E[round] by < 2^-32.  u is built exactly as the mantissa of a
// double in [1, 2) minus 1.  oracle/lioncub_oracle.py stream_uniforms
// restates it.
__device__ __forceinline__ double uniform01(uint64_t seed, int64_t e) {
  uint32_t x = (uint32_t)e * 0x9E3779B9u + (uint32_t)seed;
  x ^= (uint32_t)((uint64_t)e >> 32) * 0x85EBCA6Bu ^ (uint32_t)(seed >> 32);
  x ^= x >> 16;
  x *= 0x7FEB352Du;
  x ^= x >> 15;
  x *= 0x846CA68Bu;
  x ^= x >> 16;
  return __hiloint2double((int)(0x3FF00000u | (x >> 12)), (int)(x << 20)) - 1.0;
}

__device__ __forceinline__ float4 ld_stream(const float4* p) {
  return __ldcs(p);
}
__device__ __forceinline__ void st_stream(float4* p, float4 v) {
  __stcs(p, v);
}

// Index of the segment containing element e: start[s] <= e < start[s+1].
__device__ __forceinline__ int seg_find(const int64_t* __restrict__ start,
                                        int nseg, int64_t e) {
  int lo = 0, hi = nseg - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (__ldg(start + mid) <= e)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

// Programmatic dependent launch (Hopper+/Blackwell): the step kernels are
// launched with programmatic stream serialization so a kernel's CTAs are
// scheduled while its predecessor drains; each kernel first waits for the
// predecessor's completion (griddepcontrol.wait, a no-op without PDL).
__device__ __forceinline__ void griddep_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  // LIONCUB_PDL=0: plain stream order (A/B and diagnosis)
  static const bool pdl = [] {
    const char* e = getenv("LIONCUB_PDL");
    return !(e && e[0] == '0');
  }();
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Device view of lc_sync (kernel parameter, by value).
struct SyncD {
  uint64_t* peer[32];
  uint64_t* mine;
  uint32_t* counter;
  uint32_t* err;
  unsigned long long wait_epoch, arrive_epoch, timeout_ns;
  int P, rank;
  uint64_t* verdict;  // nullable pinned host word (lc_sync.verdict)
};

inline SyncD to_syncd(const lc_sync* s) {
  SyncD d{};
  if (!s) return d;
  for (int j = 0; j < 32; ++j) d.peer[j] = reinterpret_cast<uint64_t*>(s->peer_flags[j]);
  d.mine = s->my_flags;
  d.counter = s->counter;
  d.err = s->err;
  d.wait_epoch = s->wait_epoch;
  d.arrive_epoch = s->arrive_epoch;
  d.timeout_ns = (unsigned long long)(s->timeout_s * 1e9);
  d.P = s->P;
  d.rank = s->rank;
  d.verdict = s->verdict;
  return d;
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// A barrier wait gave up on peer j: err[0] gets LC_FLAG_BARRIER_TIMEOUT and
// err[1] bit j (the rank that never arrived, reported by CollectiveError).
__device__ __forceinline__ void sync_fail(uint32_t* err, int j) {
  atomicOr(err, (uint32_t)LC_FLAG_BARRIER_TIMEOUT);
  atomicOr(err + 1, 1u << (j & 31));
}

// Spin (one thread) until peer j's flag slot reaches `epoch`; false on
// timeout (recorded in the error words).
__device__ __forceinline__ bool wait_slot(const SyncD& s, int j, unsigned long long epoch) {
  const unsigned long long t0 = globaltimer();
  while (true) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(s.mine + j) : "memory");
    if (v >= epoch) return true;
    if (globaltimer() - t0 > s.timeout_ns) {
      sync_fail(s.err, j);
      return false;
    }
    __nanosleep(32);
  }
}

// Every CTA: wait until all P peers published s.wait_epoch (acquire).
// Returns false in every thread of the CTA if a peer timed out: the kernel
// then writes nothing (no stale words reach theta, m or a peer).
__device__ __forceinline__ bool sync_wait(const SyncD& s) {
  if (!s.wait_epoch) return true;
  const int j = threadIdx.x;
  int ok = 1;
  if (j < s.P) ok = wait_slot(s, j, s.wait_epoch);
  return __syncthreads_and(ok) != 0;
}

// The step's verdict for the host (lc_sync.verdict): every wait resolved,
// K1's flags final.  One thread.
__device__ __forceinline__ void publish_verdict(const SyncD& s, const uint32_t* flags,
                                                unsigned long long epoch, bool ok) {
  if (!s.verdict) return;
  const uint32_t f = *reinterpret_cast<const volatile uint32_t*>(flags);
  const unsigned long long v =
      (epoch << 8) | (f & 0xFu) | (ok ? 0u : (unsigned)LC_FLAG_BARRIER_TIMEOUT);
  __threadfence_system();
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(s.verdict), "l"(v) : "memory");
}

// End of a kernel: the last CTA to finish publishes s.arrive_epoch to every
// peer (each CTA fences its stores -- local and peer -- before counting).
// After a barrier timeout on this rank nothing is published, so the peers'
// waits time out too and every live rank reports the failure.
__device__ __forceinline__ void sync_arrive(const SyncD& s) {
  if (!s.arrive_epoch) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned prev = atomicAdd(s.counter, 1u);
    if (prev == gridDim.x - 1) {
      *s.counter = 0u;  // ready for the next launch of this site
      __threadfence_system();
      const uint32_t e = *reinterpret_cast<volatile uint32_t*>(s.err);
      if (e & LC_FLAG_BARRIER_TIMEOUT) return;
      for (int j = 0; j < s.P; ++j) {
        uint64_t* slot = s.peer[j] + s.rank;
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(slot), "l"(s.arrive_epoch)
                     : "memory");
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Quantizer (quant.py:127-173) over a per-segment scale table.
// ---------------------------------------------------------------------------
struct SegQ {
  const int64_t* start;
  const double* scale;
  int nseg;
  int qmax;
  const double* logs;  // per-segment log_transform scale, or null
  uint32_t qflags;     // LC_Q_*
  uint64_t seed;
};

// Cursor of the general quantizer: scale and log scale of the segment.
struct SegCursorX {
  int64_t lo = 0, hi = -1;
  double scale = 0.0, logs = 0.0;
  __device__ __forceinline__ void at(const SegQ& sq, int64_t e) {
    if (e < lo || e >= hi) {
      int s = seg_find(sq.start, sq.nseg, e);
      lo = __ldg(sq.start + s);
      hi = __ldg(sq.start + s + 1);
      scale = __ldg(sq.scale + s);
      logs = sq.logs ? __ldg(sq.logs + s) : 0.0;
    }
  }
  __device__ __forceinline__ double get(const SegQ& sq, int64_t e) {
    at(sq, e);
    return scale;
  }
};

// Every quantizer variant (quant.py:127-173): y = c or sign(c) log1p(|c|/s)
// (s > 0), v = scale * y, nearest (half-even) or stochastic rounding
// floor(v) + (u < v - floor(v)), clip to +-qmax, then no_zero: a zero q of
// a nonzero c becomes sign(c).  e: element index of the rank's flat buffer
// (the stochastic stream position).
__device__ __forceinline__ double round_x(double c, double scale, double logs, const SegQ& sq,
                                          int64_t e) {
  double y = c;
  if (logs > 0.0) {
    const double l = log1p(__ddiv_rn(fabs(c), logs));
    y = c > 0.0 ? l : (c < 0.0 ? -l : 0.0);
  }
  const double v = __dmul_rn(scale, y);
  if (sq.qflags & LC_Q_STOCHASTIC) {
    const double lo = floor(v);
    return lo + (uniform01(sq.seed, e) < __dsub_rn(v, lo) ? 1.0 : 0.0);
  }
  return rint(v);
}

__device__ __forceinline__ int quant_x(double c, const SegQ& sq, SegCursorX& cur, int64_t e) {
  cur.at(sq, e);
  double r = round_x(c, cur.scale, cur.logs, sq, e);
  r = fmin(fmax(r, -(double)sq.qmax), (double)sq.qmax);
  int q = (int)r;
  if ((sq.qflags & LC_Q_NO_ZERO) && q == 0 && c != 0.0) q = c > 0.0 ? 1 : -1;
  return q;
}

// sign(quant_x(c)) as +-1.0 / 0.0 without the int round trip (a single
// rank votes on sign(q)): the clip keeps the sign of r (qmax >= 1), rounds
// -0.0 to zero, and fmin/fmax map a NaN r to +qmax.
__device__ __forceinline__ double quant_x_sign(double c, double scale, double logs,
                                               const SegQ& sq, int64_t e) {
  const double r = round_x(c, scale, logs, sq, e);
  if (r > 0.0 || r != r) return 1.0;
  if (r < 0.0) return -1.0;
  if ((sq.qflags & LC_Q_NO_ZERO) && c != 0.0) return c > 0.0 ? 1.0 : -1.0;
  return 0.0;
}

}  // namespace lc
