// Lion Cub distributed-step kernels for B200 (sm_100a).
//
// All kernels stream fp32 state with 128-bit loads: one warp covers a tile of
// 128 consecutive elements (lane l owns elements 4l..4l+3), so the 1-bit words
// of a tile (bit b of word w = element 32w+b, quant.py:255-281 layout) are
// assembled with three shuffle-ORs across the 8 lanes that share a word.
// Math that decides a sign (c, the p-bit scale, the update) runs in float64
// with every product/sum rounded separately (no FMA contraction) so results
// equal the float64 numpy reference bit-for-bit; fp32 state is rounded once.
#include <algorithm>
#include <chrono>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>

#include "common.cuh"

namespace lc {

std::string& err_msg() {
  static thread_local std::string s;
  return s;
}

int set_err(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  err_msg() = buf;
  return code;
}

thread_local int g_grid_div = 1;  // lc_set_grid_divisor

int sm_count() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cache[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = v > 0 ? v : 148;
  }
  const int v = cache[dev] / g_grid_div;
  return v > 0 ? v : 1;
}

int resident_ctas_of(const void* kernel, int block) {
  static std::mutex mu;
  static std::map<std::tuple<int, const void*, int>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(dev, kernel, block);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, 0);
  if (per_sm < 1) per_sm = 1;
  cache.emplace(key, per_sm);
  return per_sm;
}

// Internal variants picked when the segment table asks for a quantizer
// other than nearest-rounding L1 without log map / no_zero.
constexpr int kEncQuantX = 4;    // lc_encode: QUANT_FIELDS with quant_x
constexpr int kLocalQuantX = 3;  // lc_fused_local_step: QUANT with quant_x

// Destination table: block j of a packed vector goes to p[j] (local send
// buffer, or the owner GPU's receive slot over NVLink).
struct Dst {
  void* p[LC_MAX_BLOCKS];
};

// Per-lane cache of the segment (layer) containing the current element.
struct SegCursor {
  int64_t lo = 0, hi = -1;
  double scale = 0.0;
  __device__ __forceinline__ double get(const SegQ& sq, int64_t e) {
    if (e < lo || e >= hi) {
      int s = seg_find(sq.start, sq.nseg, e);
      lo = __ldg(sq.start + s);
      hi = __ldg(sq.start + s + 1);
      scale = __ldg(sq.scale + s);
    }
    return scale;
  }
};

// q = clip(round_half_even(scale*c), +-qmax)   (quant.py:161-168)
__device__ __forceinline__ int quant_l1(double c, double scale, int qmax) {
  double r = rint(__dmul_rn(scale, c));
  r = fmin(fmax(r, -(double)qmax), (double)qmax);
  return (int)r;
}

// Pack 4 F-bit values per lane into the tile's words (element-major layout).
template <int F>
__device__ __forceinline__ void pack_store(uint32_t* __restrict__ out,
                                           int64_t t, int lane,
                                           const uint32_t st[4],
                                           int64_t nwords, bool full) {
  if constexpr (F <= 8) {
    constexpr int LPW = 8 / F;  // lanes sharing one 32-bit word
    uint32_t v = st[0] | (st[1] << F) | (st[2] << (2 * F)) | (st[3] << (3 * F));
    v <<= (4 * F) * (lane % LPW);
#pragma unroll
    for (int s = 1; s < LPW; s <<= 1) v |= __shfl_xor_sync(kFull, v, s);
    int64_t w = t * (4 * F) + lane / LPW;
    if (lane % LPW == 0 && (full || w < nwords)) out[w] = v;
  } else if constexpr (F == 16) {
    uint32_t w0 = st[0] | (st[1] << 16), w1 = st[2] | (st[3] << 16);
    int64_t w = t * 64 + 2 * lane;
    if (full) {
      *reinterpret_cast<uint2*>(out + w) = make_uint2(w0, w1);
    } else {
      if (w < nwords) out[w] = w0;
      if (w + 1 < nwords) out[w + 1] = w1;
    }
  } else {
    int64_t w = t * 128 + 4 * lane;
    if (full) {
      *reinterpret_cast<uint4*>(out + w) = make_uint4(st[0], st[1], st[2], st[3]);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (w + k < nwords) out[w + k] = st[k];
    }
  }
}

// ---------------------------------------------------------------------------
// K1: c, m', encode.  A warp owns a 1024-element super-tile (8 sub-tiles of
// 128); its 32*F packed words are staged in shared memory and leave as
// 128-byte coalesced stores to the block's destination, which is either a
// local send buffer or the owner GPU's receive slot over NVLink (Dst table:
// block j = elements [j*L, (j+1)*L) goes to dst.p[j]).
// ---------------------------------------------------------------------------
// Encode 4 consecutive elements of one lane: c and m' in float64, m' back as
// fp32, and the stored value of each element (sign bit / field).  VALID is
// false only for the last, partial sub-tile.
template <int ENC, bool MASK, class CUR>
__device__ __forceinline__ void encode4(const float ge[4], const float me[4], const bool keep[4],
                                        const bool valid[4], const Hyp& h, uint32_t fillbit,
                                        uint32_t zflag, const SegQ& sq, CUR& cur,
                                        int64_t e0, double c[4], float mn[4], uint32_t st[4],
                                        uint32_t& flag) {
  // the 4 elements usually share one layer: one segment lookup
  double qscale = 0.0;
  bool quad_in = false;
  if constexpr (ENC == LC_ENC_QUANT_FIELDS) {
    qscale = cur.get(sq, e0);
    quad_in = e0 + 3 < cur.hi;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    c[q] = lion_c(me[q], ge[q], h);
    if (MASK && !keep[q]) c[q] = 0.0;  // np.where(mask, c, 0.0)
    if (c[q] != c[q] && valid[q]) flag |= LC_FLAG_NAN;  // NaN update: the step raises
    mn[q] = lion_m(me[q], ge[q], h);
    if constexpr (ENC == LC_ENC_QUANT_FIELDS) {
      const double sc = quad_in ? qscale : cur.get(sq, e0 + q);
      st[q] = valid[q] ? (uint32_t)(quant_l1(c[q], sc, sq.qmax) + sq.qmax) : 0u;
    } else if constexpr (ENC == kEncQuantX) {
      st[q] = valid[q] ? (uint32_t)(quant_x(c[q], sq, cur, e0 + q) + sq.qmax) : 0u;
    } else if constexpr (ENC != LC_ENC_F64) {
      // sign with the zero fill; -0.0 == 0 (np.sign(-0.0) == 0); NaN -> 0
      const bool pos = c[q] > 0.0, zero = c[q] == 0.0;
      const uint32_t b = (uint32_t)pos | ((uint32_t)zero & fillbit);
      if (zero && valid[q]) flag |= zflag;
      // pad with +1 on the 1-bit wire like collectives.py:269-271
      st[q] = valid[q] ? b : (ENC == LC_ENC_SIGN1 ? 1u : 0u);
    }
  }
}

// Place one sub-tile's stored values (lane holds elements 4l..4l+3) into the
// warp's staged words for that sub-tile.
template <int F>
__device__ __forceinline__ void stage_subtile(uint32_t* sw, int lane, const uint32_t st[4]) {
  if constexpr (F <= 8) {
    constexpr int LPW = 8 / F;  // lanes sharing one 32-bit word
    uint32_t v = st[0] | (st[1] << F) | (st[2] << (2 * F)) | (st[3] << (3 * F));
    v <<= (4 * F) * (lane % LPW);
#pragma unroll
    for (int sh = 1; sh < LPW; sh <<= 1) v |= __shfl_xor_sync(kFull, v, sh);
    if (lane % LPW == 0) sw[lane / LPW] = v;
  } else if constexpr (F == 16) {
    sw[2 * lane] = st[0] | (st[1] << 16);
    sw[2 * lane + 1] = st[2] | (st[3] << 16);
  } else {
    *reinterpret_cast<uint4*>(sw + 4 * lane) = make_uint4(st[0], st[1], st[2], st[3]);
  }
}

#ifndef LC_ENC_KU
#define LC_ENC_KU 4
#endif
#ifndef LC_ENC_MINB
#define LC_ENC_MINB 2
#endif

// MPUSH (the momentum sync fused into the step, SyncPolicy layers="all"):
// m' of block j is stored into owner j's staging row for this rank
// (mst.p[j], L floats per row) instead of the local m -- the owner averages
// the P rows and stores the mean into every rank's m in k_vote_apply, so the
// all-to-all half of the sync overlaps K1's HBM stream.
template <int ENC, int F, bool MASK, bool MPUSH = false>
__global__ void __launch_bounds__(256, LC_ENC_MINB)
k_encode(const float* __restrict__ g, float* __restrict__ m,
         const uint8_t* __restrict__ mask, int64_t n, Hyp h, int fill, SegQ sq,
         Dst dst, int64_t L, int64_t eoff, int nrep, uint32_t* __restrict__ flags, SyncD sy,
         Dst mst, int64_t rot) {
  griddep_wait();
  constexpr int WPS = (ENC == LC_ENC_F64) ? 1 : 32 * F;  // words per super-tile
  constexpr int KU = LC_ENC_KU;  // sub-tiles whose loads are in flight together
  __shared__ __align__(16) uint32_t stage[8][WPS];
  // f64 c of one 128-element sub-tile per warp, re-laid out so every store
  // instruction writes 512 contiguous bytes (whole sectors: a peer's slot
  // over NVLink takes no partial-sector writes)
  __shared__ __align__(16) double cstage[ENC == LC_ENC_F64 ? 8 : 1][ENC == LC_ENC_F64 ? 128 : 2];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nsup = (n + 1023) >> 10;
  const uint32_t fillbit = fill > 0 ? 1u : 0u;
  const uint32_t zflag = fill == 0 ? (uint32_t)LC_FLAG_ZERO_SIGN : 0u;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  float4* m4 = reinterpret_cast<float4*>(m);
  uint32_t flag = 0;
  std::conditional_t<ENC == kEncQuantX, SegCursorX, SegCursor> cur;
  const bool valid_all[4] = {true, true, true, true};

  // rot: the rank's starting owner block (rank + 1), so that at any moment
  // the P ranks store into P different owners -- no incast on one owner's
  // links while the others idle (the all-to-all stays balanced).  MPUSH
  // (m' to the owners' staging rows, 4 B/param over NVLink for the remote
  // blocks) interleaves the owner blocks super-tile by super-tile instead,
  // starting at owner rank + 1: every wave of warps keeps NVLink (remote
  // blocks) and HBM (the own block) busy together, where the block-by-block
  // order ran an NVLink-bound phase and then an HBM-bound one.
  const int64_t nb = L >> 10;  // super-tiles per owner block (MPUSH: eoff == 0)
  const int64_t span = MPUSH ? (int64_t)sy.P * nb : nsup;
  for (int64_t it = gw; it < span; it += nw) {
    int64_t sidx;
    if constexpr (MPUSH) {
      const int64_t q = it / sy.P;
      const int b = (int)(it - q * sy.P);
      sidx = (int64_t)((b + sy.rank + 1) % sy.P) * nb + q;
      if (sidx >= nsup) continue;
    } else {
      sidx = it + rot;
      if (sidx >= nsup) sidx -= nsup;
    }
    const int64_t ebase = sidx << 10;
    const int64_t gbase = eoff + ebase;            // element index in the full vector
    const int j = (int)(gbase / L);
    const int64_t boff = gbase - (int64_t)j * L;  // element offset inside block j
    if (ebase + 1024 <= n) {
      // ---- fast path: a full super-tile, no per-element bounds ----
      const float4* gp = g4 + (ebase >> 2) + lane;
      float4* mp = m4 + (ebase >> 2) + lane;
#pragma unroll 1
      for (int k0 = 0; k0 < 8; k0 += KU) {
        float4 gv[KU], mv[KU];
        uchar4 mk[KU];
#pragma unroll
        for (int u = 0; u < KU; ++u) {
          gv[u] = ld_stream(gp + (k0 + u) * 32);
          mv[u] = ld_stream(mp + (k0 + u) * 32);
          if (MASK) mk[u] = *reinterpret_cast<const uchar4*>(mask + ebase + (k0 + u) * 128 + lane * 4);
        }
#pragma unroll
        for (int u = 0; u < KU; ++u) {
          const int k = k0 + u;
          const float ge[4] = {gv[u].x, gv[u].y, gv[u].z, gv[u].w};
          const float me[4] = {mv[u].x, mv[u].y, mv[u].z, mv[u].w};
          bool keep[4] = {true, true, true, true};
          if (MASK) {
            keep[0] = mk[u].x; keep[1] = mk[u].y; keep[2] = mk[u].z; keep[3] = mk[u].w;
          }
          double c[4];
          float mn[4];
          uint32_t st[4];
          encode4<ENC, MASK>(ge, me, keep, valid_all, h, fillbit, zflag, sq, cur,
                             ebase + k * 128 + lane * 4, c, mn, st, flag);
          if constexpr (MPUSH) {
            float4* sp = reinterpret_cast<float4*>(reinterpret_cast<float*>(mst.p[j]) + boff) + lane;
            st_stream(sp + k * 32, make_float4(mn[0], mn[1], mn[2], mn[3]));
          } else {
            st_stream(mp + k * 32, make_float4(mn[0], mn[1], mn[2], mn[3]));
          }
          if constexpr (ENC == LC_ENC_F64) {
            double* cs = cstage[wib];
            *reinterpret_cast<double2*>(cs + lane * 4) = make_double2(c[0], c[1]);
            *reinterpret_cast<double2*>(cs + lane * 4 + 2) = make_double2(c[2], c[3]);
            __syncwarp();
            double2* o = reinterpret_cast<double2*>(reinterpret_cast<double*>(dst.p[j]) + boff +
                                                    k * 128);
            o[lane] = reinterpret_cast<const double2*>(cs)[lane];
            o[32 + lane] = reinterpret_cast<const double2*>(cs)[32 + lane];
            __syncwarp();
          } else {
            stage_subtile<F>(&stage[wib][k * 4 * F], lane, st);
          }
        }
      }
    } else {
      // ---- tail super-tile: per-element bounds ----
#pragma unroll 1
      for (int k = 0; k < 8; ++k) {
        const int64_t e0 = ebase + k * 128 + lane * 4;
        if (ebase + k * 128 >= n) {  // whole sub-tile past the end (warp-uniform)
          if (ENC != LC_ENC_F64)
            for (int w = lane; w < 4 * F; w += 32) stage[wib][k * 4 * F + w] = 0u;
          continue;
        }
        float ge[4], me[4];
        bool valid[4], keep[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          valid[q] = e0 + q < n;
          ge[q] = valid[q] ? g[e0 + q] : 0.f;
          me[q] = valid[q] ? m[e0 + q] : 0.f;
          keep[q] = MASK ? (valid[q] ? mask[e0 + q] != 0 : true) : true;
        }
        double c[4];
        float mn[4];
        uint32_t st[4];
        encode4<ENC, MASK>(ge, me, keep, valid, h, fillbit, zflag, sq, cur, e0, c, mn, st, flag);
        float* mdst = m + e0;
        if constexpr (MPUSH) mdst = reinterpret_cast<float*>(mst.p[j]) + boff + k * 128 + lane * 4;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (valid[q]) mdst[q] = mn[q];
        if constexpr (ENC == LC_ENC_F64) {
          double* o = reinterpret_cast<double*>(dst.p[j]) + boff + k * 128 + lane * 4;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (valid[q]) o[q] = c[q];
        } else {
          stage_subtile<F>(&stage[wib][k * 4 * F], lane, st);
        }
      }
    }
    if constexpr (ENC != LC_ENC_F64) {
      __syncwarp();
      const int64_t rem = n - ebase;
      const int nwv = rem >= 1024 ? WPS : (int)((rem * F + 31) / 32);
      // owner-block mode: block j's destination; replicate mode (nrep > 0):
      // the same words to every destination (an allgather of the payload)
      const int nd = nrep > 0 ? nrep : 1;
      for (int q = 0; q < nd; ++q) {
        uint32_t* d = reinterpret_cast<uint32_t*>(dst.p[nrep > 0 ? q : j]) + (boff >> 5) * F;
        if (nwv == WPS && (WPS % 128) == 0) {
          for (int w = lane * 4; w < WPS; w += 128)
            *reinterpret_cast<uint4*>(d + w) = *reinterpret_cast<const uint4*>(&stage[wib][w]);
        } else {
          for (int w = lane; w < nwv; w += 32) d[w] = stage[wib][w];
        }
      }
      __syncwarp();
    }
  }
  if (flag) atomicOr(flags, flag);
  sync_arrive(sy);
}

// ---------------------------------------------------------------------------
// K5: theta update from (sign bits, optional nonzero bits).  A warp owns a
// 1024-element super-tile: lane i fetches word i of its 32 voted words with
// one coalesced 128-byte load from the word's owner -- the local gather
// buffer, or the owner GPU's vote output over NVLink (src table indexed by
// owner block, wpb words per block) -- then sub-tile k takes its 4 words by
// shuffle.  theta streams with KU sub-tiles of float4 loads in flight.
// ---------------------------------------------------------------------------
template <bool NZ>
__global__ void __launch_bounds__(256, 3)
k_apply_update(float* __restrict__ theta, int64_t n, Dst sb, Dst nzb, int64_t wpb,
               int64_t woff, double lr, double wd, SyncD sy) {
  constexpr int KU = 4;
  griddep_wait();
  if (!sync_wait(sy)) return;  // a peer never voted: theta stays untouched
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nsup = (n + 1023) >> 10;
  const int64_t nwords = (n + 31) >> 5;
  float4* th4 = reinterpret_cast<float4*>(theta);
  // voted words of super-tile sidx (lane i: word i), fetched one super-tile
  // ahead so a remote owner's NVLink latency overlaps the theta stream
  auto fetch = [&](int64_t sidx, uint32_t& sw_, uint32_t& zw_) {
    const int64_t w = sidx * 32 + lane;
    sw_ = 0u;
    zw_ = ~0u;
    if (sidx < nsup && w < nwords) {
      const int64_t wg = woff + w;  // word index in the full vector
      const int j = (int)(wg / wpb);
      sw_ = __ldcs(reinterpret_cast<const uint32_t*>(sb.p[j]) + wg);
      if (NZ) zw_ = __ldcs(reinterpret_cast<const uint32_t*>(nzb.p[j]) + wg);
    }
  };
  uint32_t nxw, nxz;
  fetch(gw, nxw, nxz);
  for (int64_t sidx = gw; sidx < nsup; sidx += nw) {
    const uint32_t myw = nxw, myz = nxz;
    fetch(sidx + nw, nxw, nxz);
#pragma unroll 1
    for (int k0 = 0; k0 < 8; k0 += KU) {
      float4 tv[KU];
#pragma unroll
      for (int u = 0; u < KU; ++u) {
        const int64_t t = sidx * 8 + k0 + u;
        if ((t + 1) * 128 <= n) tv[u] = ld_stream(th4 + t * 32 + lane);
      }
#pragma unroll
      for (int u = 0; u < KU; ++u) {
        const int k = k0 + u;
        const int64_t t = sidx * 8 + k;
        const uint32_t sw = __shfl_sync(kFull, myw, 4 * k + (lane >> 3));
        const uint32_t zw = NZ ? __shfl_sync(kFull, myz, 4 * k + (lane >> 3)) : ~0u;
        if (t * 128 >= n) continue;  // warp-uniform
        const int sh = 4 * (lane & 7);
        const uint32_t sn = (sw >> sh) & 0xF, zn = (zw >> sh) & 0xF;
        double sg[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          sg[q] = ((zn >> q) & 1) ? (((sn >> q) & 1) ? 1.0 : -1.0) : 0.0;
        if ((t + 1) * 128 <= n) {
          float4 v = tv[u];
          v.x = lion_theta(v.x, sg[0], lr, wd);
          v.y = lion_theta(v.y, sg[1], lr, wd);
          v.z = lion_theta(v.z, sg[2], lr, wd);
          v.w = lion_theta(v.w, sg[3], lr, wd);
          st_stream(th4 + t * 32 + lane, v);
        } else {
          const int64_t e0 = t * 128 + lane * 4;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (e0 + q < n) theta[e0 + q] = lion_theta(theta[e0 + q], sg[q], lr, wd);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Fused single-rank step (P == 1): one pass, theta/m/g in, theta'/m' out.
// ---------------------------------------------------------------------------
#ifndef LC_FUSED_U
#define LC_FUSED_U 2
#endif
#ifndef LC_FUSED_MINB
#define LC_FUSED_MINB 3
#endif
// Quantized modes (L1 / general quantizer): one tile in flight per warp at
// 4 CTAs/SM beats two at 3 (GPT-2, P = 1, fused kernel: L1 5-bit 0.460 ->
// 0.441 ms, Q_inf stochastic 0.633 -> 0.599 ms; sign modes unchanged).
#ifndef LC_FUSED_QU
#define LC_FUSED_QU 1
#endif
#ifndef LC_FUSED_QMINB
#define LC_FUSED_QMINB 4
#endif
constexpr bool fused_quant(int mode) { return mode == LC_LOCAL_QUANT || mode == kLocalQuantX; }
constexpr int fused_u(int mode) { return fused_quant(mode) ? LC_FUSED_QU : LC_FUSED_U; }

template <int MODE, bool MASK, bool METRICS, int U>
__global__ void __launch_bounds__(256, fused_quant(MODE) ? LC_FUSED_QMINB : LC_FUSED_MINB)
k_fused_local(float* __restrict__ theta, float* __restrict__ m,
              const float* __restrict__ g, const uint8_t* __restrict__ mask,
              int64_t n, Hyp h, double lr, double wd, int fill, SegQ sq,
              uint32_t* __restrict__ sbits, uint32_t* __restrict__ nzbits,
              uint32_t* __restrict__ tbits, uint32_t* __restrict__ flags) {
  griddep_wait();
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t ntiles = (n + 127) >> 7, nfull = n >> 7;
  const int64_t nwords = (n + 31) >> 5;
  const bool ternary = fill == 0;
  const double fillv = fill > 0 ? 1.0 : (fill < 0 ? -1.0 : 0.0);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  float4* m4 = reinterpret_cast<float4*>(m);
  float4* th4 = reinterpret_cast<float4*>(theta);
  uint32_t flag = 0;
  std::conditional_t<MODE == kLocalQuantX, SegCursorX, SegCursor> cur;
  for (int64_t t0 = gw; t0 < ntiles; t0 += nw * U) {
    float4 gv[U], mv[U], tv[U];
    uchar4 mk[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int64_t t = t0 + u * nw;
      if (t < nfull) {
        gv[u] = ld_stream(g4 + t * 32 + lane);
        mv[u] = ld_stream(m4 + t * 32 + lane);
        tv[u] = ld_stream(th4 + t * 32 + lane);
        if (MASK) mk[u] = *reinterpret_cast<const uchar4*>(mask + t * 128 + lane * 4);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t t = t0 + u * nw;
      if (t >= ntiles) break;
      const bool full = t < nfull;
      const int64_t e0 = t * 128 + lane * 4;
      float ge[4], me[4], te[4];
      bool valid[4], keep[4];
      if (full) {
        ge[0] = gv[u].x; ge[1] = gv[u].y; ge[2] = gv[u].z; ge[3] = gv[u].w;
        me[0] = mv[u].x; me[1] = mv[u].y; me[2] = mv[u].z; me[3] = mv[u].w;
        te[0] = tv[u].x; te[1] = tv[u].y; te[2] = tv[u].z; te[3] = tv[u].w;
#pragma unroll
        for (int k = 0; k < 4; ++k) valid[k] = true;
        if (MASK) {
          keep[0] = mk[u].x; keep[1] = mk[u].y; keep[2] = mk[u].z; keep[3] = mk[u].w;
        }
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          valid[k] = e0 + k < n;
          ge[k] = valid[k] ? g[e0 + k] : 0.f;
          me[k] = valid[k] ? m[e0 + k] : 0.f;
          te[k] = valid[k] ? theta[e0 + k] : 0.f;
          keep[k] = MASK ? (valid[k] ? mask[e0 + k] != 0 : true) : true;
        }
      }
      float mn[4], tn[4];
      uint32_t sbit[4], nzb[4], tb[4];
      // the lane's 4 elements usually share one layer: one segment lookup
      double qscale = 0.0;
      bool quad_in = false;
      if constexpr (MODE == LC_LOCAL_QUANT || MODE == kLocalQuantX) {
        qscale = cur.get(sq, e0);
        quad_in = e0 + 3 < cur.hi;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        double c = lion_c(me[k], ge[k], h);
        if (MASK && !keep[k]) c = 0.0;
        mn[k] = lion_m(me[k], ge[k], h);
        double agg;  // the single-rank aggregate the vote signs
        if constexpr (MODE == LC_LOCAL_QUANT) {
          // one rank's vote is sign(q): rint(v) != 0 iff |v| > 0.5 (half-even),
          // and clipping keeps the sign, so only v = scale*c is needed (a NaN
          // v gives -1 like clip(rint(NaN)) = -qmax)
          const double v = __dmul_rn(quad_in ? qscale : cur.get(sq, e0 + k), c);
          agg = valid[k] ? (v > 0.5 ? 1.0 : (v >= -0.5 ? 0.0 : -1.0)) : 1.0;
        } else if constexpr (MODE == kLocalQuantX) {
          agg = 1.0;
          if (valid[k]) {
            if (!quad_in) cur.at(sq, e0 + k);
            agg = quant_x_sign(c, cur.scale, cur.logs, sq, e0 + k);
          }
        } else {
          agg = c;
        }
        double s;
        bool zero = false;
        if (agg > 0.0) {
          s = 1.0;
        } else if (agg < 0.0) {
          s = -1.0;
        } else if (agg == 0.0) {
          zero = MODE != LC_LOCAL_BINARY;
          if (MODE == LC_LOCAL_BINARY && ternary && valid[k]) flag |= LC_FLAG_ZERO_SIGN;
          s = fillv;
        } else {  // NaN: theta' = NaN like numpy's float path; the step raises
          s = __longlong_as_double(0x7ff8000000000000ll);
          if (valid[k]) flag |= LC_FLAG_NAN;
        }
        tn[k] = lion_theta(te[k], s, lr, wd);
        sbit[k] = s > 0.0 ? 1u : 0u;
        nzb[k] = s != 0.0 ? 1u : 0u;
        tb[k] = (zero && valid[k]) ? 1u : 0u;
      }
      if (full) {
        st_stream(m4 + t * 32 + lane, make_float4(mn[0], mn[1], mn[2], mn[3]));
        st_stream(th4 + t * 32 + lane, make_float4(tn[0], tn[1], tn[2], tn[3]));
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (valid[k]) {
            m[e0 + k] = mn[k];
            theta[e0 + k] = tn[k];
          }
      }
      if (METRICS) {
        if (sbits) pack_store<1>(sbits, t, lane, sbit, nwords, full);
        if (nzbits) pack_store<1>(nzbits, t, lane, nzb, nwords, full);
        if (tbits) pack_store<1>(tbits, t, lane, tb, nwords, full);
      }
    }
  }
  if (flag) atomicOr(flags, flag);
}

// ---------------------------------------------------------------------------
// K4: 1-bit majority over P packed chunks, bit-sliced counting.  Each thread
// votes 4 words (uint4 loads of every rank's chunk) and writes the result to
// `nout` destinations: the local gather buffer (NCCL path) or every rank's
// gather buffer over NVLink (the allgather fused into the vote).
//   sum_mode 0: compressed1bit -- a tie in exact-ternary mode is an error
//               (collectives.py:290-293).
//   sum_mode 1: sum-of-signs (direct, bits=1) -- the tally IS the p-bit sum
//               2k-P; a zero sum gives a zero update in exact-ternary mode.
// ---------------------------------------------------------------------------
struct VoteOut {
  Dst v, nz, tie;
  int nout;  // > 0: that many destinations; -1: p[0] is an NVLS multicast address
};

// NVLS: one store to a multicast address is replicated by the NVSwitch into
// the bound buffer of every GPU (the allgather as a single store).
__device__ __forceinline__ void mc_st4(uint32_t* mc, uint4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};"
               ::"l"(mc), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void mc_st1(uint32_t* mc, uint32_t v) {
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(mc), "r"(v) : "memory");
}

__device__ __forceinline__ void vote_store(const VoteOut& o, int64_t i, uint4 v, uint4 nz,
                                           uint4 tie) {
  if (o.nout < 0) {
    mc_st4(reinterpret_cast<uint32_t*>(o.v.p[0]) + i, v);
    if (o.nz.p[0]) mc_st4(reinterpret_cast<uint32_t*>(o.nz.p[0]) + i, nz);
    if (o.tie.p[0]) mc_st4(reinterpret_cast<uint32_t*>(o.tie.p[0]) + i, tie);
    return;
  }
  for (int k = 0; k < o.nout; ++k) {
    *reinterpret_cast<uint4*>(reinterpret_cast<uint32_t*>(o.v.p[k]) + i) = v;
    if (o.nz.p[0]) *reinterpret_cast<uint4*>(reinterpret_cast<uint32_t*>(o.nz.p[k]) + i) = nz;
    if (o.tie.p[0]) *reinterpret_cast<uint4*>(reinterpret_cast<uint32_t*>(o.tie.p[k]) + i) = tie;
  }
}

__device__ __forceinline__ void vote_store1(const VoteOut& o, int k, int64_t i, uint32_t v,
                                            uint32_t nz, uint32_t tie) {
  if (o.nout < 0) {
    mc_st1(reinterpret_cast<uint32_t*>(o.v.p[0]) + i, v);
    if (o.nz.p[0]) mc_st1(reinterpret_cast<uint32_t*>(o.nz.p[0]) + i, nz);
    if (o.tie.p[0]) mc_st1(reinterpret_cast<uint32_t*>(o.tie.p[0]) + i, tie);
    return;
  }
  reinterpret_cast<uint32_t*>(o.v.p[k])[i] = v;
  if (o.nz.p[0]) reinterpret_cast<uint32_t*>(o.nz.p[k])[i] = nz;
  if (o.tie.p[0]) reinterpret_cast<uint32_t*>(o.tie.p[k])[i] = tie;
}

template <int NP>
__device__ __forceinline__ void vote_word(uint32_t planes[NP], int P, int T, uint32_t fillmask,
                                          uint32_t vm, int fill, int sum_mode, uint32_t& v,
                                          uint32_t& nz, uint32_t& tie, uint32_t& flag) {
  uint32_t gt = 0u, eq = ~0u;
#pragma unroll
  for (int p = NP - 1; p >= 0; --p) {
    uint32_t pl = planes[p];
    if ((T >> p) & 1) {
      eq &= pl;
    } else {
      gt |= eq & pl;
      eq &= ~pl;
    }
  }
  if (P & 1) {  // count > (P-1)/2 is a strict majority; no ties possible
    v = gt;
    eq = 0u;
  } else {
    v = gt | (eq & fillmask);
    if (fill == 0 && sum_mode == 0 && (eq & vm)) flag |= LC_FLAG_TIE_TERNARY;
  }
  tie = eq & vm;
  nz = ~eq & vm;
}

template <int NP>
__global__ void __launch_bounds__(256)
k_vote_bits(const uint32_t* __restrict__ recv, int P, int64_t cw, int64_t n_valid,
            int fill, int sum_mode, VoteOut out, uint32_t* __restrict__ flags, SyncD sy) {
  griddep_wait();
  if (!sync_wait(sy)) {  // a peer's words never arrived: vote nothing
    sync_arrive(sy);
    return;
  }
  const int T = P >> 1;
  const uint32_t fillmask = fill > 0 ? ~0u : 0u;
  uint32_t flag = 0;
  const int64_t nq = cw >> 2;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq;
       q += (int64_t)gridDim.x * blockDim.x) {
    uint32_t pl[4][NP];
#pragma unroll
    for (int w = 0; w < 4; ++w)
#pragma unroll
      for (int p = 0; p < NP; ++p) pl[w][p] = 0u;
    for (int j = 0; j < P; ++j) {
      uint4 x = __ldcs(reinterpret_cast<const uint4*>(recv + (int64_t)j * cw) + q);
      uint32_t xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        uint32_t carry = xs[w];
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          uint32_t t = pl[w][p] & carry;
          pl[w][p] ^= carry;
          carry = t;
        }
      }
    }
    uint32_t v[4], nz[4], tie[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      int64_t rem = n_valid - (4 * q + w) * 32;
      uint32_t vm = rem >= 32 ? ~0u : (rem <= 0 ? 0u : ((1u << rem) - 1u));
      vote_word<NP>(pl[w], P, T, fillmask, vm, fill, sum_mode, v[w], nz[w], tie[w], flag);
    }
    vote_store(out, 4 * q, make_uint4(v[0], v[1], v[2], v[3]),
               make_uint4(nz[0], nz[1], nz[2], nz[3]), make_uint4(tie[0], tie[1], tie[2], tie[3]));
  }
  if (flag) atomicOr(flags, flag);
  sync_arrive(sy);
}

// ---------------------------------------------------------------------------
// K4+K5 fused (peer-memory path): the grid votes the owner block in
// warp-sized units and pushes the voted words into every rank's gather
// buffer; the warp completing the last unit publishes epoch e2.  The same
// grid then updates theta in work items handed out by a counter, this
// rank's own block first, each warp waiting only for the owner of the block
// it is about to read (so the update of already-voted blocks overlaps the
// slowest owner's vote).  Both phases are work-counter driven, so nothing
// waits on a CTA that is not resident (round 2: a static split deadlocked
// when another stream's kernel held a few SM slots).
// ---------------------------------------------------------------------------
struct ApplyArgs {
  float* theta;
  int64_t n;
  const uint32_t* sb;   // local gather buffer (all blocks land here)
  const uint32_t* nzb;  // nullable
  double lr, wd;
  int64_t blk_words;    // words per owner block (cw)
  int64_t chunk;        // super-tiles per work item of the update phase
};

#ifndef LC_VOTE_SHARE
#define LC_VOTE_SHARE 8  // P >= 4: the first 1/LC_VOTE_SHARE of the CTAs to start vote
#endif

// The momentum sync fused into the step (the owner half of
// allreduce_mean_f32, collectives.py:319-344): this owner's P staged rows of
// m' (stage + r*L, written by every rank's K1 in MPUSH mode) are summed in
// float64 in rank order, divided once, rounded once to fp32 and stored into
// every rank's momentum block (out.p[k]).  Chunks are taken from a work
// counter by every CTA once its vote / theta role is done.
struct MeanArgs {
  const float* stage;  // null: no sync this step
  Dst out;             // out.p[k]: rank k's momentum + owner offset
  int64_t L;           // staging row stride (floats)
  int64_t cnt;         // valid elements of this owner's block
  unsigned int* work;  // zeroed chunk counter
};

constexpr int kMeanChunk = 8192;  // elements per work item (256 threads x 8 float4)

__device__ __forceinline__ float4 mean_of(const double acc[4], double dp) {
  return make_float4(__double2float_rn(__ddiv_rn(acc[0], dp)), __double2float_rn(__ddiv_rn(acc[1], dp)),
                     __double2float_rn(__ddiv_rn(acc[2], dp)), __double2float_rn(__ddiv_rn(acc[3], dp)));
}

// Owner mean of one chunk: each thread holds kMeanILP quads; for every rank
// row their loads are issued together (the row order of the float64 sum is
// kept), then the fp32 means go to every rank's momentum.
template <int kMeanILP>  // float4 quads per thread whose row loads are in flight together
__device__ __forceinline__ void mean_chunk(const MeanArgs& ma, int P, int64_t c0, int64_t q1,
                                           double dp) {
  const int64_t step = 4 * (int64_t)blockDim.x;
  for (int64_t base = c0 + 4 * (int64_t)threadIdx.x; base < q1; base += step * kMeanILP) {
    double acc[kMeanILP][4];
    bool on[kMeanILP];
#pragma unroll
    for (int u = 0; u < kMeanILP; ++u) on[u] = base + u * step < q1;
    for (int r = 0; r < P; ++r) {
      const float* row = ma.stage + (int64_t)r * ma.L;
      float4 x[kMeanILP];
#pragma unroll
      for (int u = 0; u < kMeanILP; ++u)
        if (on[u]) x[u] = __ldcs(reinterpret_cast<const float4*>(row + base + u * step));
#pragma unroll
      for (int u = 0; u < kMeanILP; ++u) {
        if (!on[u]) continue;
        if (r == 0) {
          acc[u][0] = x[u].x; acc[u][1] = x[u].y; acc[u][2] = x[u].z; acc[u][3] = x[u].w;
        } else {
          acc[u][0] = __dadd_rn(acc[u][0], (double)x[u].x);
          acc[u][1] = __dadd_rn(acc[u][1], (double)x[u].y);
          acc[u][2] = __dadd_rn(acc[u][2], (double)x[u].z);
          acc[u][3] = __dadd_rn(acc[u][3], (double)x[u].w);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kMeanILP; ++u) {
      if (!on[u]) continue;
      const float4 v = mean_of(acc[u], dp);
      const int64_t i = base + u * step;
      for (int k = 0; k < P; ++k)
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(ma.out.p[k]) + i) = v;
    }
  }
}

template <int ILP>
__device__ void mean_role(const MeanArgs& ma, int P) {
  __shared__ long long chunk;
  const double dp = (double)P;
  while (true) {
    __syncthreads();
    if (threadIdx.x == 0) chunk = (long long)atomicAdd(ma.work, 1u);
    __syncthreads();
    const int64_t c0 = (int64_t)chunk * kMeanChunk;
    if (c0 >= ma.cnt) break;
    const int64_t c1 = c0 + kMeanChunk < ma.cnt ? c0 + kMeanChunk : ma.cnt;
    const int64_t q1 = c0 + ((c1 - c0) & ~(int64_t)3);
    mean_chunk<ILP>(ma, P, c0, q1, dp);
    for (int64_t i = q1 + threadIdx.x; i < c1; i += blockDim.x) {  // ragged tail
      double acc = (double)ma.stage[i];
      for (int r = 1; r < P; ++r) acc = __dadd_rn(acc, (double)ma.stage[(int64_t)r * ma.L + i]);
      const float v = __double2float_rn(__ddiv_rn(acc, dp));
      for (int k = 0; k < P; ++k) reinterpret_cast<float*>(ma.out.p[k])[i] = v;
    }
  }
}

// The fused sync's owner mean as its own lean kernel, run on a side stream
// CONCURRENTLY with k_vote_apply (whose grid is capped so both are
// resident): the NVLink-store-bound mean overlaps the HBM-bound theta update.
// It needs only every rank's K1 (sy.wait_epoch = e1).
__global__ void __launch_bounds__(256, 4)
k_sync_mean(SyncD sy, MeanArgs ma, int P) {
  griddep_wait();
  if (!sync_wait(sy)) return;  // a peer's staged rows never arrived: no mean
  mean_role<2>(ma, P);
}

#ifndef LC_VA_CHUNK
#define LC_VA_CHUNK 8    // max super-tiles per work item of the update phase
#endif
#ifndef LC_VA_ITEMS
#define LC_VA_ITEMS 32768   // work items per launch the chunk size aims for (GPT-2 size: 4 super-tiles)
#endif

#ifndef LC_VA_UNIT
#define LC_VA_UNIT 256
#endif
constexpr int kVoteUnitQuads = LC_VA_UNIT;  // max uint4 word quads per vote unit (32K elements)

// The update phase's work counter (sy.counter[1]) is reset by the last CTA
// to finish its update (sy.counter[2] counts them), so the next launch on
// the same sync site -- ordered after this grid -- starts from zero.
__device__ __forceinline__ void va_retire(const SyncD& sy) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(sy.counter + 2, 1u) == gridDim.x - 1) {
      sy.counter[1] = 0u;
      sy.counter[2] = 0u;
      sy.counter[3] = 0u;
      sy.counter[4] = 0u;
      __threadfence();
    }
  }
}

// Vote units of k_vote_apply.  Claims warp-sized units (the next claim in
// flight while a unit is voted) until none is left, then counts its units
// done with one system fence; the warp whose count completes the block
// publishes e2.  Returns false (units exhausted).
template <int NP>
__device__ __forceinline__ void va_vote_quad(const uint32_t* __restrict__ recv, int P, int T,
                                             int64_t cw, int64_t n_valid, int fill,
                                             uint32_t fillmask, int sum_mode, const VoteOut& out,
                                             int64_t q0, int64_t q1, uint32_t& flag) {
  // two quads per lane with their P row loads in flight together
  const bool on1 = q1 < (cw >> 2);
  uint32_t pl[2][4][NP];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int w = 0; w < 4; ++w)
#pragma unroll
      for (int pp = 0; pp < NP; ++pp) pl[h][w][pp] = 0u;
#pragma unroll 2
  for (int j = 0; j < P; ++j) {
    const uint4* row = reinterpret_cast<const uint4*>(recv + (int64_t)j * cw);
    const uint4 x0 = __ldcs(row + q0);
    const uint4 x1 = on1 ? __ldcs(row + q1) : make_uint4(0u, 0u, 0u, 0u);
    const uint32_t xs[2][4] = {{x0.x, x0.y, x0.z, x0.w}, {x1.x, x1.y, x1.z, x1.w}};
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        uint32_t carry = xs[h][w];
#pragma unroll
        for (int pp = 0; pp < NP; ++pp) {
          const uint32_t t = pl[h][w][pp] & carry;
          pl[h][w][pp] ^= carry;
          carry = t;
        }
      }
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (h == 1 && !on1) break;
    const int64_t q = h ? q1 : q0;
    uint32_t v[4], nz[4], tie[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const int64_t rem = n_valid - (4 * q + w) * 32;
      const uint32_t vm = rem >= 32 ? ~0u : (rem <= 0 ? 0u : ((1u << rem) - 1u));
      vote_word<NP>(pl[h][w], P, T, fillmask, vm, fill, sum_mode, v[w], nz[w], tie[w], flag);
    }
    vote_store(out, 4 * q, make_uint4(v[0], v[1], v[2], v[3]),
               make_uint4(nz[0], nz[1], nz[2], nz[3]), make_uint4(tie[0], tie[1], tie[2], tie[3]));
  }
}

template <int NP>
__device__ __forceinline__ bool va_vote_units(const uint32_t* __restrict__ recv, int P, int T,
                                              int64_t cw, int64_t n_valid, int fill,
                                              uint32_t fillmask, int sum_mode, const VoteOut& out,
                                              uint32_t* flags, const SyncD& sy, int64_t nunits,
                                              int64_t unit, int lane) {
  const int64_t nq = cw >> 2;
  unsigned int* vclaim = sy.counter + 3;
  unsigned int* vdone = sy.counter;
  unsigned int u = 0u, ahead = 0u, mine = 0u;
  if (lane == 0) u = atomicAdd(vclaim, 1u);
  u = __shfl_sync(kFull, u, 0);
  if ((int64_t)u < nunits && lane == 0) ahead = atomicAdd(vclaim, 1u);
  uint32_t flag = 0;
  while ((int64_t)u < nunits) {
    const int64_t qe = min(nq, ((int64_t)u + 1) * unit);
    for (int64_t q = (int64_t)u * unit + lane; q < qe; q += 64)
      va_vote_quad<NP>(recv, P, T, cw, n_valid, fill, fillmask, sum_mode, out, q,
                       q + 32 < qe ? q + 32 : nq, flag);
    ++mine;
    u = __shfl_sync(kFull, ahead, 0);
    if ((int64_t)u < nunits && lane == 0) ahead = atomicAdd(vclaim, 1u);
  }
  if (flag) atomicOr(flags, flag);
  __syncwarp();
  if (mine && lane == 0) {
    __threadfence_system();  // this warp's stores (local and peers) first
    if (atomicAdd(vdone, mine) + mine == (unsigned int)nunits) {
      *vdone = 0u;  // ready for the next launch of this site
      __threadfence_system();
      const uint32_t e = *reinterpret_cast<volatile uint32_t*>(sy.err);
      if (!(e & LC_FLAG_BARRIER_TIMEOUT)) {
        for (int j = 0; j < sy.P; ++j)
          asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(sy.peer[j] + sy.rank),
                       "l"(sy.arrive_epoch) : "memory");
      }
    }
  }
  __syncwarp();
  return false;
}


// WIDE: the grid has the GPU to itself -- 3 CTAs/SM (80 registers), 8 theta
// sub-tiles in flight per warp.  Otherwise (capped beside the fused sync's
// mean kernel, or running the mean itself) 4 CTAs/SM at 64 registers and 4
// sub-tiles, so 2 vote CTAs + 2 mean CTAs fit an SM's register file.
// Measured (4 x B200): 1.1B vote/update 1.52 ms WIDE vs 1.56; the 7e9 fused
// sync step at P = 2 50.4 ms narrow vs 54.4 ms WIDE (mean CTAs starved).
template <int NP, bool NZ, bool MEAN, bool WIDE>
__global__ void __launch_bounds__(256, WIDE ? 3 : 4)
k_vote_apply(const uint32_t* __restrict__ recv, int P, int64_t cw, int64_t n_valid, int fill,
             int sum_mode, const __grid_constant__ VoteOut out, uint32_t* __restrict__ flags,
             const __grid_constant__ SyncD sy, ApplyArgs a,
             MeanArgs ma) {
  griddep_wait();
  if (!sync_wait(sy)) {  // a peer's words never arrived: no vote, no theta update
    if (blockIdx.x == 0 && threadIdx.x == 0) publish_verdict(sy, flags, sy.arrive_epoch, false);
    va_retire(sy);
    return;
  }
  const int T = P >> 1;
  const uint32_t fillmask = fill > 0 ? ~0u : 0u;
  const int lane = threadIdx.x & 31;
  // ---- 1. the owner vote (as k_vote_bits) in warp-sized units taken from a
  // counter (sy.counter[3]); the warp whose finished units complete the
  // block publishes e2 (sy.counter[0] counts them).  At P >= 4 the first
  // 1/LC_VOTE_SHARE of the CTAs TO START (a ticket, sy.counter[4] -- not
  // blockIdx) vote while the others begin the theta update of this rank's
  // own block, voting those words in-warp, so the vote's NVLink pushes
  // overlap the HBM-bound update.  Voters are CTAs that are running, and
  // units are handed out dynamically, so e2 never waits for a CTA that is
  // not resident (another stream's kernel may hold some of the SMs).  At
  // P <= 3 every CTA votes first (measured faster for 1.1B at P = 2: the
  // pushed half is too large for a fraction of the SMs) ----
  __shared__ int s_voter;
  const int share = P >= 4 ? LC_VOTE_SHARE : 1;
  const unsigned int nvote = max(1u, gridDim.x / share);
  if (threadIdx.x == 0) s_voter = atomicAdd(sy.counter + 4, 1u) < nvote;
  __syncthreads();
  const int64_t nq = cw >> 2;
  // at most kVoteUnitQuads per unit, and ~4 units per voter warp so a small
  // block's vote (the critical path to e2) spreads over every voter
  int64_t unit = nq / ((int64_t)nvote * (blockDim.x >> 5) * 4);
  unit = unit < 32 ? 32 : (unit > kVoteUnitQuads ? kVoteUnitQuads : (unit & ~(int64_t)31));
  if (s_voter)
    va_vote_units<NP>(recv, P, T, cw, n_valid, fill, fillmask, sum_mode, out, flags, sy,
                      (nq + unit - 1) / unit, unit, lane);
  if (sy.verdict && blockIdx.x == 0 && threadIdx.x == 0) {
    // the host's verdict once every owner (this one included: its vote
    // flags are final) has published its block -- the waits left in the
    // update below then all succeed at once
    bool ok = true;
    for (int j = 0; j < P; ++j) ok = wait_slot(sy, j, sy.arrive_epoch) && ok;
    publish_verdict(sy, flags, sy.arrive_epoch, ok);
  }
  // ---- 2. theta update.  Warps take work items of up to LC_VA_CHUNK
  // super-tiles from a counter (sy.counter[1]) in rotated order -- this
  // rank's own block first (voted in-warp at P >= 4: no wait), so the peers'
  // blocks are usually out by the time the items reach them -- waiting per
  // owner block for its e2 ----
  constexpr int KU = WIDE ? 8 : 4;  // theta sub-tiles in flight per warp
  const int64_t CH = a.chunk;
  const int64_t nsup = (a.n + 1023) >> 10;
  const int64_t nwords = (a.n + 31) >> 5;
  float4* th4 = reinterpret_cast<float4*>(a.theta);
  uint32_t ready = 0u;  // owners whose voted block this warp has seen land
  uint32_t bad = 0u;    // owners whose barrier timed out
  auto fetch = [&](int64_t sidx, uint32_t& sw_, uint32_t& zw_) {
    sw_ = 0u;
    zw_ = ~0u;
    if (sidx >= nsup) return;
    const int j = (int)((sidx * 32) / a.blk_words);  // owner of this super-tile
    if (j == sy.rank && share > 1) {  // own block: vote this word from the P rows
      const int64_t wl = sidx * 32 + lane - (int64_t)j * a.blk_words;  // word in my block
      uint32_t pl[NP];
#pragma unroll
      for (int pp = 0; pp < NP; ++pp) pl[pp] = 0u;
      if (wl < cw) {
        for (int r = 0; r < P; ++r) {
          uint32_t carry = __ldcs(recv + (int64_t)r * cw + wl);
#pragma unroll
          for (int pp = 0; pp < NP; ++pp) {
            const uint32_t t = pl[pp] & carry;
            pl[pp] ^= carry;
            carry = t;
          }
        }
      }
      const int64_t rem = n_valid - wl * 32;
      const uint32_t vm = rem >= 32 ? ~0u : (rem <= 0 ? 0u : ((1u << rem) - 1u));
      uint32_t v, nz, tie, fl = 0;
      vote_word<NP>(pl, P, T, fillmask, vm, fill, sum_mode, v, nz, tie, fl);
      sw_ = v;
      if (NZ) zw_ = nz;
      return;
    }
    if (!(((ready | bad) >> j) & 1u)) {
      int ok = 1;
      if (lane == 0) ok = wait_slot(sy, j, sy.arrive_epoch);
      ok = __shfl_sync(kFull, ok, 0);
      if (ok) ready |= 1u << j;
      else bad |= 1u << j;  // owner j never published: its block is not updated
    }
    const int64_t w = sidx * 32 + lane;
    if (w < nwords) {
      sw_ = __ldcv(a.sb + w);
      if (NZ) zw_ = __ldcv(a.nzb + w);
    }
  };
  int64_t rot = (int64_t)sy.rank * a.blk_words / 32;  // blk_words % 32 == 0
  if (rot >= nsup) rot = 0;
  auto at = [&](int64_t i) {
    if (i >= nsup) return nsup;  // past the end: fetch() returns nothing
    const int64_t s = i + rot;
    return s >= nsup ? s - nsup : s;
  };
  auto update = [&](int64_t sidx, uint32_t myw, uint32_t myz) {
#pragma unroll 1
    for (int k0 = 0; k0 < 8; k0 += KU) {
      float4 tv[KU];
#pragma unroll
      for (int u = 0; u < KU; ++u) {
        const int64_t t = sidx * 8 + k0 + u;
        if ((t + 1) * 128 <= a.n) tv[u] = ld_stream(th4 + t * 32 + lane);
      }
#pragma unroll
      for (int u = 0; u < KU; ++u) {
        const int k = k0 + u;
        const int64_t t = sidx * 8 + k;
        const uint32_t sw = __shfl_sync(kFull, myw, 4 * k + (lane >> 3));
        const uint32_t zw = NZ ? __shfl_sync(kFull, myz, 4 * k + (lane >> 3)) : ~0u;
        if (t * 128 >= a.n) continue;  // warp-uniform
        const int sh = 4 * (lane & 7);
        const uint32_t sn = (sw >> sh) & 0xF, zn = (zw >> sh) & 0xF;
        double sg[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          sg[q] = ((zn >> q) & 1) ? (((sn >> q) & 1) ? 1.0 : -1.0) : 0.0;
        if ((t + 1) * 128 <= a.n) {
          float4 v = tv[u];
          v.x = lion_theta(v.x, sg[0], a.lr, a.wd);
          v.y = lion_theta(v.y, sg[1], a.lr, a.wd);
          v.z = lion_theta(v.z, sg[2], a.lr, a.wd);
          v.w = lion_theta(v.w, sg[3], a.lr, a.wd);
          st_stream(th4 + t * 32 + lane, v);
        } else {
          const int64_t e0 = t * 128 + lane * 4;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (e0 + q < a.n) a.theta[e0 + q] = lion_theta(a.theta[e0 + q], sg[q], a.lr, a.wd);
        }
      }
    }
  };
  // positions (item, c) in the order the counter hands items out; the voted
  // words of the next position are fetched one super-tile ahead and the next
  // item's index is requested one item ahead, so neither latency is exposed
  unsigned int* work = sy.counter + 1;
  const int64_t nitems = (nsup + CH - 1) / CH;
  unsigned int cur = 0u, ahead = 0u;
  if (lane == 0) cur = atomicAdd(work, 1u);
  cur = __shfl_sync(kFull, cur, 0);
  if (lane == 0) ahead = atomicAdd(work, 1u);
  int64_t c = 0;
  uint32_t nxw, nxz;
  fetch((int64_t)cur < nitems ? at((int64_t)cur * CH) : nsup, nxw, nxz);
  while ((int64_t)cur < nitems) {
    const int64_t sidx = at((int64_t)cur * CH + c);
    const uint32_t myw = nxw, myz = nxz;
    unsigned int ncur = cur;
    int64_t nc = c + 1;
    if (nc == CH) {
      ncur = __shfl_sync(kFull, ahead, 0);
      nc = 0;
      if (lane == 0) ahead = atomicAdd(work, 1u);
    }
    fetch((int64_t)ncur < nitems ? at((int64_t)ncur * CH + nc) : nsup, nxw, nxz);
    if (sidx < nsup && !((bad >> (int)((sidx * 32) / a.blk_words)) & 1u))  // bad: stale words
      update(sidx, myw, myz);
    cur = ncur;
    c = nc;
  }
  va_retire(sy);
  // every CTA whose theta share is done joins the fused momentum mean
  // (needs only e1: the staged rows are complete even if an owner's vote timed out)
  if constexpr (MEAN) {
    if (ma.stage) mean_role<4>(ma, P);
  }
}

// ---------------------------------------------------------------------------
// K6: p-bit field sums -> signed aggregate -> sign words (+ ties, values).
// `rows` partial-sum rows of the owner block are added first (1 after an
// NCCL reduce-scatter; P when peers wrote their fields over NVLink).  Each
// lane reads one input word (E = 32/F elements); F lanes form a sign word.
// ---------------------------------------------------------------------------
template <int F>
__global__ void __launch_bounds__(256)
k_fields_vote(const uint32_t* __restrict__ sums, int rows, int64_t row_stride, int64_t n,
              int P, int offset, int binary, int fill, VoteOut out,
              int64_t* __restrict__ values, SyncD sy) {
  griddep_wait();
  if (!sync_wait(sy)) {
    sync_arrive(sy);
    return;
  }
  constexpr int E = 32 / F;
  constexpr uint32_t FM = (F == 32) ? 0xffffffffu : ((1u << F) - 1u);
  const int lane = threadIdx.x & 31;
  const int64_t nin = (n * F + 31) / 32;
  const int64_t nout = (n + 31) / 32;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nchunks = (nin + 31) / 32;
  for (int64_t ch = gw; ch < nchunks; ch += nw) {
    const int64_t i = ch * 32 + lane;
    uint32_t w = 0u;
    if (i < nin)
      for (int r = 0; r < rows; ++r) w += __ldcs(sums + (int64_t)r * row_stride + i);
    uint32_t pos = 0u, zer = 0u, val = 0u;
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const int64_t e = i * E + k;
      if (e < n) {
        const int64_t cnt = (int64_t)((w >> (F * k)) & FM);
        const int64_t s = binary ? 2 * cnt - P : cnt - (int64_t)P * offset;
        pos |= (uint32_t)(s > 0) << k;
        zer |= (uint32_t)(s == 0) << k;
        val |= 1u << k;
        if (values) values[e] = s;
      }
    }
    const int shift = (int)(i % F) * E;
    if (E < 32) {
      pos <<= shift;
      zer <<= shift;
      val <<= shift;
    }
#pragma unroll
    for (int s = 1; s < F; s <<= 1) {
      pos |= __shfl_xor_sync(kFull, pos, s);
      zer |= __shfl_xor_sync(kFull, zer, s);
      val |= __shfl_xor_sync(kFull, val, s);
    }
    const int64_t o = i / F;
    if ((lane % F) == 0 && o < nout) {
      const uint32_t v = pos | (fill > 0 ? zer : 0u);
      const int nk = out.nout < 0 ? 1 : out.nout;
      for (int k = 0; k < nk; ++k) vote_store1(out, k, o, v, ~zer & val, zer & val);
    }
  }
  sync_arrive(sy);
}

// K6 without per-element values (the step path): one thread per output sign
// word -- it adds its F input words over the rows with 128-bit loads and
// decodes 32 fields in registers (no shuffles).
template <int F>
__global__ void __launch_bounds__(256)
k_fields_vote_words(const uint32_t* __restrict__ sums, int rows, int64_t row_stride, int64_t n,
                    int P, int offset, int binary, int fill, VoteOut out, SyncD sy) {
  griddep_wait();
  if (!sync_wait(sy)) {
    sync_arrive(sy);
    return;
  }
  constexpr int E = 32 / F;  // fields per input word
  constexpr uint32_t FM = (F == 32) ? 0xffffffffu : ((1u << F) - 1u);
  const int64_t nout = (n + 31) / 32;
  const int64_t nin = (n * F + 31) / 32;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < nout;
       o += (int64_t)gridDim.x * blockDim.x) {
    uint32_t w[F];
#pragma unroll
    for (int k = 0; k < F; ++k) w[k] = 0u;
    const int64_t i0 = o * F;
    const bool vec = (F >= 4) && (i0 + F <= nin);
    for (int r = 0; r < rows; ++r) {
      const uint32_t* src = sums + (int64_t)r * row_stride + i0;
      if (vec) {
#pragma unroll
        for (int k = 0; k < F; k += 4) {
          const uint4 x = __ldcs(reinterpret_cast<const uint4*>(src + k));
          w[k] += x.x; w[k + 1] += x.y; w[k + 2] += x.z; w[k + 3] += x.w;
        }
      } else {
#pragma unroll
        for (int k = 0; k < F; ++k)
          if (i0 + k < nin) w[k] += __ldcs(src + k);
      }
    }
    uint32_t pos = 0u, zer = 0u;
#pragma unroll
    for (int b = 0; b < 32; ++b) {
      const int64_t cnt = (int64_t)((w[b / E] >> (F * (b % E))) & FM);
      const int64_t sv = binary ? 2 * cnt - P : cnt - (int64_t)P * offset;
      pos |= (uint32_t)(sv > 0) << b;
      zer |= (uint32_t)(sv == 0) << b;
    }
    const int64_t rem = n - o * 32;
    const uint32_t val = rem >= 32 ? ~0u : ((1u << rem) - 1u);
    zer &= val;
    const int nk = out.nout < 0 ? 1 : out.nout;
    for (int k = 0; k < nk; ++k) vote_store1(out, k, o, pos | (fill > 0 ? zer : 0u), ~zer & val, zer);
  }
  sync_arrive(sy);
}

// ---------------------------------------------------------------------------
// Full-precision arm: rank-ordered float64 sum (flat or binomial tree).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
k_f64_sum_vote(const double* __restrict__ recv, int P, int64_t len, int64_t stride, int tree,
               int fill, VoteOut out, double* __restrict__ values, SyncD sy) {
  griddep_wait();
  if (!sync_wait(sy)) {
    sync_arrive(sy);
    return;
  }
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nwords = (len + 31) / 32;
  for (int64_t w = gw; w < nwords; w += nw) {
    const int64_t e = w * 32 + lane;
    const bool valid = e < len;
    double tot = 0.0;
    if (valid) {
      if (!tree) {
        tot = recv[e];
        for (int j = 1; j < P; ++j) tot = __dadd_rn(tot, recv[(int64_t)j * stride + e]);
      } else {
        double acc[64];
        for (int j = 0; j < P; ++j) acc[j] = recv[(int64_t)j * stride + e];
        for (int mk = 1; mk < P; mk <<= 1)
          for (int r = 0; r + mk < P; r += 2 * mk) acc[r] = __dadd_rn(acc[r], acc[r + mk]);
        tot = acc[0];
      }
      if (values) values[e] = tot;
    }
    const uint32_t pb = __ballot_sync(kFull, valid && tot > 0.0);
    const uint32_t zb = __ballot_sync(kFull, valid && tot == 0.0);
    const uint32_t vb = __ballot_sync(kFull, valid);
    if (lane < (out.nout < 0 ? 1 : out.nout))
      vote_store1(out, lane, w, pb | (fill > 0 ? zb : 0u), ~zb & vb, zb);
  }
  sync_arrive(sy);
}

// K7: momentum mean, float64 accumulation in rank order, one fp32 rounding.
__global__ void __launch_bounds__(256)
k_mean_f32(const float* __restrict__ recv, int P, int64_t len, int64_t stride,
           float* __restrict__ out) {
  const double dp = (double)P;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len;
       i += (int64_t)gridDim.x * blockDim.x) {
    double acc = (double)__ldcs(recv + i);
    for (int j = 1; j < P; ++j) acc = __dadd_rn(acc, (double)__ldcs(recv + (int64_t)j * stride + i));
    out[i] = __double2float_rn(__ddiv_rn(acc, dp));
  }
}

__global__ void k_compute_c(const float* __restrict__ g, const float* __restrict__ m,
                            const uint8_t* __restrict__ mask, int64_t n, Hyp h,
                            double* __restrict__ c) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = lion_c(m[i], g[i], h);
    if (mask && !mask[i]) v = 0.0;
    c[i] = v;
  }
}

__global__ void k_count_bits_seg(const uint32_t* __restrict__ bits,
                                 const int64_t* __restrict__ start, int nseg,
                                 int64_t* __restrict__ counts) {
  const int64_t n = start[nseg];
  const int64_t nwords = (n + 31) / 32;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwords;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t b = bits[w];
    int64_t e = w * 32;
    int64_t end = e + 32 < n ? e + 32 : n;
    if (end - e < 32) b &= (1u << (end - e)) - 1u;
    if (!b) continue;
    int s = seg_find(start, nseg, e);
    while (e < end) {
      int64_t se = start[s + 1];
      int64_t hi = se < end ? se : end;
      int lo_bit = (int)(e - w * 32), hi_bit = (int)(hi - w * 32);
      uint32_t msk = (hi_bit >= 32 ? ~0u : ((1u << hi_bit) - 1u)) & ~((1u << lo_bit) - 1u);
      int cnt = __popc(b & msk);
      if (cnt) atomicAdd(reinterpret_cast<unsigned long long*>(counts + s),
                         (unsigned long long)cnt);
      e = hi;
      ++s;
    }
  }
}

__global__ void k_bits_to_sign(const uint32_t* __restrict__ sb,
                               const uint32_t* __restrict__ nzb, int64_t n,
                               int8_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t bit = (sb[i >> 5] >> (i & 31)) & 1u;
    int8_t v = bit ? 1 : -1;
    if (nzb && !((nzb[i >> 5] >> (i & 31)) & 1u)) v = 0;
    out[i] = v;
  }
}

template <int F>
__global__ void k_pack_i64(const int64_t* __restrict__ v, int64_t n, int offset,
                           int binary, uint32_t* __restrict__ out,
                           uint32_t* __restrict__ flags) {
  constexpr int E = 32 / F;
  const int64_t nwords = (n * F + 31) / 32;
  const uint64_t lim = (F == 32) ? 0xffffffffull : ((1ull << F) - 1ull);
  uint32_t flag = 0;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwords;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t word = 0;
#pragma unroll
    for (int k = 0; k < E; ++k) {
      int64_t e = w * E + k;
      if (e < n) {
        int64_t x = v[e];
        int64_t st;
        if (binary) {
          if (x != 1 && x != -1) flag |= LC_FLAG_RANGE;
          st = (x + 1) >> 1;
        } else {
          st = x + offset;
        }
        if (st < 0 || (uint64_t)st > lim) {
          flag |= LC_FLAG_RANGE;
          st = 0;
        }
        word |= (uint32_t)st << (F * k % 32);
      }
    }
    out[w] = word;
  }
  if (flag) atomicOr(flags, flag);
}

template <int F>
__global__ void k_fields_decode(const uint32_t* __restrict__ sums, int64_t n, int P,
                                int offset, int binary, int64_t* __restrict__ out) {
  constexpr int E = 32 / F;
  constexpr uint32_t FM = (F == 32) ? 0xffffffffu : ((1u << F) - 1u);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t cnt = (int64_t)((sums[e / E] >> (F * (int)(e % E))) & FM);
    out[e] = binary ? 2 * cnt - P : cnt - (int64_t)P * offset;
  }
}

__global__ void k_sign_pack_f64(const double* __restrict__ c, int64_t n, int fill,
                                uint32_t* __restrict__ out, uint32_t* __restrict__ flags) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nwords = (n + 31) / 32;
  uint32_t flag = 0;
  for (int64_t w = gw; w < nwords; w += nw) {
    int64_t e = w * 32 + lane;
    bool valid = e < n;
    double x = valid ? c[e] : 1.0;
    bool bit;
    if (x > 0.0) bit = true;
    else if (x < 0.0) bit = false;
    else if (x == 0.0) {
      bit = fill > 0;
      if (fill == 0) flag |= LC_FLAG_ZERO_SIGN;
    } else {
      bit = false;
      flag |= LC_FLAG_NAN;
    }
    uint32_t b = __ballot_sync(kFull, bit || !valid);
    if (lane == 0) out[w] = b;
  }
  if (flag) atomicOr(flags, flag);
}

// Exact-ternary pre-flight of the binary paths: zero signs of c (and the
// sign words for the owner tie check), without materialising c.
__global__ void k_sign_check(const float* __restrict__ g, const float* __restrict__ m,
                             const uint8_t* __restrict__ mask, int64_t n, Hyp h,
                             uint32_t* __restrict__ out, uint32_t* __restrict__ flags) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nwords = (n + 31) / 32;
  bool zero = false;
  for (int64_t w = gw; w < nwords; w += nw) {
    const int64_t e = w * 32 + lane;
    bool pos = true;  // padding past n: +1 like the wire
    if (e < n) {
      double c = lion_c(__ldcs(m + e), __ldcs(g + e), h);
      if (mask && !mask[e]) c = 0.0;
      pos = c > 0.0;
      zero |= c == 0.0;
    }
    const uint32_t b = __ballot_sync(kFull, pos);
    if (out && lane == 0) out[w] = b;
  }
  if (__any_sync(kFull, zero) && lane == 0) atomicOr(flags, (uint32_t)LC_FLAG_ZERO_SIGN);
}

struct Rows {
  const uint32_t* p[64];
};

__global__ void k_sum_rows(Rows rows, int P, int64_t count, uint32_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t s = 0;
    for (int j = 0; j < P; ++j) s += rows.p[j][i];
    out[i] = s;
  }
}

// ---------------------------------------------------------------------------
// K5v: vote + theta update for the allgather exchange (peer-memory path,
// P <= 4 by default).  K1 in replicate mode stored every rank's sign words
// into row `rank` of every rank's receive rows, so each rank holds all P
// rows of the whole vector: a warp owns a 1024-element super-tile, lane i
// counts word i over the P rows (bit-sliced, the same count the owner's K4
// makes), votes it, and sub-tile k takes its 4 voted words by shuffle.  No
// owner hop and no voted-word broadcast: one in-kernel barrier per step.
// ---------------------------------------------------------------------------
#ifndef LC_VU_KU
#define LC_VU_KU 4
#endif
#ifndef LC_VU_MINB
#define LC_VU_MINB 3
#endif

template <int NP, bool NZ>
__global__ void __launch_bounds__(256, LC_VU_MINB)
k_vote_update(const uint32_t* __restrict__ rows, int64_t stride, int P, float* __restrict__ theta,
              int64_t n, int fill, int sum_mode, double lr, double wd,
              uint32_t* __restrict__ flags, SyncD sy) {
  constexpr int KU = LC_VU_KU;  // theta sub-tiles in flight per batch
  griddep_wait();
  const bool synced = sync_wait(sy);
  // every wait of the step is behind us: the host may check it now
  if (blockIdx.x == 0 && threadIdx.x == 0) publish_verdict(sy, flags, sy.wait_epoch, synced);
  if (!synced) return;  // a peer's rows never arrived: theta untouched
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nsup = (n + 1023) >> 10;
  const int64_t nwords = (n + 31) >> 5;
  const uint32_t fillmask = fill > 0 ? ~0u : 0u;
  const int T = P >> 1;
  float4* th4 = reinterpret_cast<float4*>(theta);
  uint32_t flag = 0;
  for (int64_t sidx = gw; sidx < nsup; sidx += nw) {
    const int64_t eb = sidx << 10;
    const bool full = eb + 1024 <= n;
    float4 tv[KU];  // the first batch of theta in flight with the words
    if (full) {
#pragma unroll
      for (int k = 0; k < KU; ++k) tv[k] = ld_stream(th4 + (eb >> 2) + k * 32 + lane);
    }
    const int64_t w = sidx * 32 + lane;
    uint32_t myw = 0u, myz = ~0u;
    if (w < nwords) {
      uint32_t pl[NP];
#pragma unroll
      for (int pp = 0; pp < NP; ++pp) pl[pp] = 0u;
      for (int s4 = 0; s4 < P; s4 += 4) {
        uint32_t x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) x[u] = s4 + u < P ? __ldcg(rows + (int64_t)(s4 + u) * stride + w) : 0u;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          uint32_t carry = x[u];
#pragma unroll
          for (int pp = 0; pp < NP; ++pp) {
            const uint32_t t = pl[pp] & carry;
            pl[pp] ^= carry;
            carry = t;
          }
        }
      }
      const int64_t rem = n - w * 32;
      const uint32_t vm = rem >= 32 ? ~0u : ((1u << rem) - 1u);
      uint32_t tie;
      vote_word<NP>(pl, P, T, fillmask, vm, fill, sum_mode, myw, myz, tie, flag);
    }
#pragma unroll
    for (int k0 = 0; k0 < 8; k0 += KU) {
      if (k0 > 0 && full) {
#pragma unroll
        for (int u = 0; u < KU; ++u) tv[u] = ld_stream(th4 + (eb >> 2) + (k0 + u) * 32 + lane);
      }
#pragma unroll
      for (int u = 0; u < KU; ++u) {
        const int k = k0 + u;
        const int64_t t = sidx * 8 + k;
        const uint32_t sw = __shfl_sync(kFull, myw, 4 * k + (lane >> 3));
        const uint32_t zw = NZ ? __shfl_sync(kFull, myz, 4 * k + (lane >> 3)) : ~0u;
        const int sh = 4 * (lane & 7);
        const uint32_t sn = (sw >> sh) & 0xF, zn = (zw >> sh) & 0xF;
        double sg[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) sg[q] = ((zn >> q) & 1) ? (((sn >> q) & 1) ? 1.0 : -1.0) : 0.0;
        if (full) {
          float4 v = tv[u];
          v.x = lion_theta(v.x, sg[0], lr, wd);
          v.y = lion_theta(v.y, sg[1], lr, wd);
          v.z = lion_theta(v.z, sg[2], lr, wd);
          v.w = lion_theta(v.w, sg[3], lr, wd);
          st_stream(th4 + t * 32 + lane, v);
        } else if (t * 128 < n) {
          const int64_t e0 = t * 128 + lane * 4;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (e0 + q < n) theta[e0 + q] = lion_theta(theta[e0 + q], sg[q], lr, wd);
        }
      }
    }
  }
  if (flag) atomicOr(flags, flag);
}

// An empty launch that still takes part in the in-kernel barriers: a rank
// whose share of a phase is empty (an owner block past the end of a short
// vector) must publish its epoch all the same, or its peers time out.
__global__ void k_sync_only(SyncD sy) {
  griddep_wait();
  sync_wait(sy);
  sync_arrive(sy);
}

}  // namespace lc

// ===========================================================================
// C ABI
// ===========================================================================
using namespace lc;

namespace {

constexpr int kBlock = 256;

Hyp to_hyp(const lc_hyper* h) { return Hyp{h->beta1, h->one_minus_beta1, h->beta2, h->one_minus_beta2}; }

SegQ to_segq(const lc_segments* s) {
  SegQ q{nullptr, nullptr, 0, 0, nullptr, 0u, 0ull};
  if (s) {
    q.start = s->start;
    q.scale = s->scale;
    q.nseg = s->nseg;
    q.qmax = s->qmax;
    q.logs = s->log_scale;
    q.qflags = s->qflags;
    q.seed = s->seed;
  }
  return q;
}

// The segment table asks for a quantizer beyond nearest-rounding L1.
bool needs_quant_x(const lc_segments* s) { return s && (s->log_scale || s->qflags); }

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int generic_grid(int64_t n) {
  int64_t b = (n + kBlock - 1) / kBlock;
  int64_t cap = (int64_t)sm_count() * 8;
  if (b > cap) b = cap;
  return b < 1 ? 1 : (int)b;
}

thread_local SyncD g_sync{};     // sync of the encode launch being dispatched
thread_local int64_t g_eoff = 0;  // element offset of the encode launch
thread_local int g_nrep = 0;      // replicate-mode destinations (0: owner blocks)
thread_local bool g_mpush = false;  // m' -> owners' staging rows (g_mst)
thread_local Dst g_mst{};
thread_local int64_t g_rot = 0;     // starting super-tile of the encode launch

// Owner-block exchanges start each rank at owner (rank + 1) % P.
int64_t encode_rotation(const lc_sync* sync, int64_t n, int64_t L, int64_t eoff, bool rep) {
  if (!sync || sync->P < 2 || rep || eoff != 0) return 0;
  const int64_t nsup = (n + 1023) >> 10;
  if (nsup < 1) return 0;
  return ((int64_t)((sync->rank + 1) % sync->P) * (L >> 10)) % nsup;
}

template <int ENC, int F, bool MASK>
int launch_encode(const float* g, float* m, const uint8_t* mask, int64_t n, Hyp h,
                  int fill, SegQ sq, const Dst& dst, int64_t L, uint32_t* flags,
                  cudaStream_t st) {
  int64_t nsup = (n + 1023) >> 10;
  if constexpr (ENC == LC_ENC_SIGN1) {
    if (g_mpush) {
      auto kern = k_encode<ENC, F, MASK, true>;
      int grid = stream_grid(kern, kBlock, nsup, kBlock / 32);
      LC_CUDA_TRY(launch_pdl(kern, grid, kBlock, 0, st, g, m, mask, n, h, fill, sq, dst, L,
                             g_eoff, g_nrep, flags, g_sync, g_mst, g_rot));
      LC_LAUNCH_CHECK();
      return LC_OK;
    }
  }
  auto kern = k_encode<ENC, F, MASK, false>;
  int grid = stream_grid(kern, kBlock, nsup, kBlock / 32);
  LC_CUDA_TRY(launch_pdl(kern, grid, kBlock, 0, st, g, m, mask, n, h, fill, sq, dst, L, g_eoff,
                         g_nrep, flags, g_sync, g_mst, g_rot));
  LC_LAUNCH_CHECK();
  return LC_OK;
}

template <int ENC, int F>
int dispatch_mask(const float* g, float* m, const uint8_t* mask, int64_t n, Hyp h,
                  int fill, SegQ sq, const Dst& dst, int64_t L, uint32_t* flags,
                  cudaStream_t st) {
  if (mask) return launch_encode<ENC, F, true>(g, m, mask, n, h, fill, sq, dst, L, flags, st);
  return launch_encode<ENC, F, false>(g, m, mask, n, h, fill, sq, dst, L, flags, st);
}

template <int ENC>
int dispatch_fields(int F, const float* g, float* m, const uint8_t* mask, int64_t n,
                    Hyp h, int fill, SegQ sq, const Dst& dst, int64_t L, uint32_t* flags,
                    cudaStream_t st) {
  switch (F) {
    case 1: return dispatch_mask<ENC, 1>(g, m, mask, n, h, fill, sq, dst, L, flags, st);
    case 2: return dispatch_mask<ENC, 2>(g, m, mask, n, h, fill, sq, dst, L, flags, st);
    case 4: return dispatch_mask<ENC, 4>(g, m, mask, n, h, fill, sq, dst, L, flags, st);
    case 8: return dispatch_mask<ENC, 8>(g, m, mask, n, h, fill, sq, dst, L, flags, st);
    case 16: return dispatch_mask<ENC, 16>(g, m, mask, n, h, fill, sq, dst, L, flags, st);
    case 32: return dispatch_mask<ENC, 32>(g, m, mask, n, h, fill, sq, dst, L, flags, st);
    default: return set_err(LC_E_ARG, "field_bits must be 1,2,4,8,16,32 (got %d)", F);
  }
}

// Nothing to compute, but the launch's barrier role stays (k_sync_only).
int sync_only(const lc_sync* sync, void* stream) {
  if (!sync || (!sync->wait_epoch && !sync->arrive_epoch)) return LC_OK;
  LC_CUDA_TRY(launch_pdl(k_sync_only, 1, 32, 0, reinterpret_cast<cudaStream_t>(stream),
                         to_syncd(sync)));
  LC_LAUNCH_CHECK();
  return LC_OK;
}

// Build a Dst table from a host array of nd pointers (nd <= LC_MAX_BLOCKS).
bool make_dst(Dst& d, void* const* ptrs, int nd) {
  if (nd < 1 || nd > LC_MAX_BLOCKS || !ptrs) return false;
  for (int i = 0; i < LC_MAX_BLOCKS; ++i) d.p[i] = i < nd ? ptrs[i] : nullptr;
  for (int i = 0; i < nd; ++i)
    if (!d.p[i]) return false;
  return true;
}

}  // namespace

extern "C" {

int lc_abi_version(void) { return LIONCUB_ABI_VERSION; }

int lc_wait_verdict(const uint64_t* word, uint64_t epoch, double timeout_s, uint32_t* status) {
  if (!word || !status) return set_err(LC_E_ARG, "lc_wait_verdict: null pointer");
  const auto t0 = std::chrono::steady_clock::now();
  for (uint32_t spin = 0;; ++spin) {
    const uint64_t v = __atomic_load_n(word, __ATOMIC_ACQUIRE);
    if ((v >> 8) >= epoch) {
      *status = (uint32_t)(v & 0xFFu);
      return LC_OK;
    }
    if ((spin & 255u) == 255u) {
      const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (dt > timeout_s) return set_err(LC_E_COLLECTIVE, "lc_wait_verdict: no verdict before the timeout");
      if (dt > 1e-3) std::this_thread::yield();
    }
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  }
}

const char* lc_last_error(void) { return err_msg().c_str(); }

int lc_set_grid_divisor(int divisor) {
  if (divisor < 1 || divisor > 1024) return set_err(LC_E_ARG, "lc_set_grid_divisor: divisor in [1,1024]");
  g_grid_div = divisor;
  return LC_OK;
}

int lc_device_sm_count(int device) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess)
    return set_err(LC_E_CUDA, "cudaDeviceGetAttribute failed");
  return v;
}

int lc_encode(const float* g, float* m, const uint8_t* mask, int64_t n,
              const lc_hyper* hp, int fill, int enc, int field_bits,
              const lc_segments* segs, void* const* dst, int32_t nblocks, int64_t L,
              int64_t eoff, uint32_t* flags, const lc_sync* sync, void* stream) {
  if (n < 0 || !hp || !flags) return set_err(LC_E_ARG, "lc_encode: bad arguments");
  if (n == 0) return sync_only(sync, stream);
  if (!g || !m) return set_err(LC_E_ARG, "lc_encode: null pointer");
  if (!aligned16(g) || !aligned16(m)) return set_err(LC_E_ARG, "lc_encode: g/m must be 16-byte aligned");
  const bool rep = (enc & LC_ENC_REPLICATE) != 0;
  enc &= ~LC_ENC_REPLICATE;
  if (rep && (enc != LC_ENC_SIGN1 || L < eoff + n))
    return set_err(LC_E_ARG, "lc_encode: replicate mode is 1-bit only and L must cover [eoff, eoff+n)");
  if (L <= 0 || (L % 1024) != 0 || (!rep && (int64_t)nblocks * L < eoff + n) || eoff < 0 ||
      (eoff % 1024) != 0)
    return set_err(LC_E_ARG, "lc_encode: blocks (multiple of 1024) must cover [eoff, eoff+n), eoff % 1024 == 0");
  Dst d;
  if (!make_dst(d, dst, nblocks)) return set_err(LC_E_ARG, "lc_encode: bad destination table");
  g_nrep = rep ? nblocks : 0;
  g_mpush = false;
  g_rot = encode_rotation(sync, n, L, eoff, rep);
  Hyp h = to_hyp(hp);
  SegQ sq = to_segq(segs);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  g_sync = to_syncd(sync);
  g_eoff = eoff;
  switch (enc) {
    case LC_ENC_SIGN1:
      return dispatch_mask<LC_ENC_SIGN1, 1>(g, m, mask, n, h, fill, sq, d, L, flags, st);
    case LC_ENC_SIGN_FIELDS:
      return dispatch_fields<LC_ENC_SIGN_FIELDS>(field_bits, g, m, mask, n, h, fill, sq, d, L, flags, st);
    case LC_ENC_QUANT_FIELDS:
      if (!segs || !segs->start || !segs->scale || segs->nseg < 1)
        return set_err(LC_E_ARG, "lc_encode: quant needs a segment table with scales");
      if (field_bits < 2) return set_err(LC_E_ARG, "lc_encode: quant fields need >= 2 bits");
      if (needs_quant_x(segs))
        return dispatch_fields<kEncQuantX>(field_bits, g, m, mask, n, h, fill, sq, d, L, flags, st);
      return dispatch_fields<LC_ENC_QUANT_FIELDS>(field_bits, g, m, mask, n, h, fill, sq, d, L, flags, st);
    case LC_ENC_F64:
      return dispatch_mask<LC_ENC_F64, 1>(g, m, mask, n, h, fill, sq, d, L, flags, st);
    default:
      return set_err(LC_E_ARG, "lc_encode: unknown encoding %d", enc);
  }
}

int lc_encode_sync(const float* g, float* m, const uint8_t* mask, int64_t n,
                   const lc_hyper* hp, int fill, void* const* dst, int32_t nblocks, int64_t L,
                   uint32_t* flags, const lc_sync* sync, void* const* mstage, void* stream) {
  Dst ms;
  if (!mstage || !make_dst(ms, mstage, nblocks) || !dst || nblocks < 1)
    return set_err(LC_E_ARG, "lc_encode_sync: one staging row per owner block required");
  for (int j = 0; j < nblocks; ++j)
    if ((reinterpret_cast<uintptr_t>(ms.p[j]) & 15u) != 0)
      return set_err(LC_E_ARG, "lc_encode_sync: staging rows must be 16-byte aligned");
  // the plain 1-bit encode, with m' routed to the owners' staging rows
  if (n < 0 || !hp || !flags) return set_err(LC_E_ARG, "lc_encode_sync: bad arguments");
  if (n == 0) return sync_only(sync, stream);
  if (!g || !m || !aligned16(g) || !aligned16(m))
    return set_err(LC_E_ARG, "lc_encode_sync: g/m must be 16-byte aligned");
  if (L <= 0 || (L % 1024) != 0 || (int64_t)nblocks * L < n)
    return set_err(LC_E_ARG, "lc_encode_sync: blocks (multiple of 1024) must cover n");
  Dst d;
  if (!make_dst(d, dst, nblocks)) return set_err(LC_E_ARG, "lc_encode_sync: bad destination table");
  if (!sync || sync->P != nblocks || sync->rank < 0 || sync->rank >= nblocks)
    return set_err(LC_E_ARG, "lc_encode_sync: sync required, with P == nblocks (it orders the owner blocks)");
  g_nrep = 0;
  g_eoff = 0;
  g_sync = to_syncd(sync);
  g_mst = ms;
  g_mpush = true;
  g_rot = encode_rotation(sync, n, L, 0, false);
  const int rc = dispatch_mask<LC_ENC_SIGN1, 1>(g, m, mask, n, to_hyp(hp), fill, to_segq(nullptr), d,
                                                 L, flags, reinterpret_cast<cudaStream_t>(stream));
  g_mpush = false;
  return rc;
}

int lc_apply_update(float* theta, int64_t n, void* const* sign_bits, void* const* nz_bits,
                    int32_t nsrc, int64_t wpb, int64_t woff, double lr, double wd,
                    const lc_sync* sync, void* stream) {
  if (n < 0) return set_err(LC_E_ARG, "lc_apply_update: n < 0");
  if (n == 0) return sync_only(sync, stream);
  Dst sb, zb;
  if (!theta || !make_dst(sb, sign_bits, nsrc) || (nz_bits && !make_dst(zb, nz_bits, nsrc)))
    return set_err(LC_E_ARG, "lc_apply_update: bad pointers / source table");
  if (wpb <= 0 || woff < 0 || (int64_t)nsrc * wpb * 32 < woff * 32 + n)
    return set_err(LC_E_ARG, "lc_apply_update: source blocks do not cover [woff*32, woff*32+n)");
  if (!aligned16(theta)) return set_err(LC_E_ARG, "lc_apply_update: theta must be 16-byte aligned");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int64_t nsup = (n + 1023) >> 10;
  if (nz_bits) {
    auto kern = k_apply_update<true>;
    int grid = stream_grid(kern, kBlock, nsup, kBlock / 32);
    LC_CUDA_TRY(launch_pdl(kern, grid, kBlock, 0, st, theta, n, sb, zb, wpb, woff, lr, wd,
                           to_syncd(sync)));
  } else {
    auto kern = k_apply_update<false>;
    int grid = stream_grid(kern, kBlock, nsup, kBlock / 32);
    LC_CUDA_TRY(launch_pdl(kern, grid, kBlock, 0, st, theta, n, sb, sb, wpb, woff, lr, wd,
                           to_syncd(sync)));
  }
  LC_LAUNCH_CHECK();
  return LC_OK;
}

int lc_fused_local_step(float* theta, float* m, const float* g, const uint8_t* mask,
                        int64_t n, const lc_hyper* hp, int fill, int mode,
                        const lc_segments* segs, uint32_t* sign_bits,
                        uint32_t* nz_bits, uint32_t* tie_bits, uint32_t* flags,
                        void* stream) {
  if (n < 0 || !hp || !flags) return set_err(LC_E_ARG, "lc_fused_local_step: bad arguments");
  if (n == 0) return LC_OK;
  if (!theta || !m || !g) return set_err(LC_E_ARG, "lc_fused_local_step: null pointer");
  if (!aligned16(theta) || !aligned16(m) || !aligned16(g))
    return set_err(LC_E_ARG, "lc_fused_local_step: theta/m/g must be 16-byte aligned");
  if (mode == LC_LOCAL_QUANT && (!segs || !segs->scale || !segs->start))
    return set_err(LC_E_ARG, "lc_fused_local_step: quant needs segment scales");
  Hyp h = to_hyp(hp);
  SegQ sq = to_segq(segs);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool metrics = sign_bits || nz_bits || tie_bits;
  const int64_t ntiles = (n + 127) >> 7;
#define LC_FUSED(MODE, MASK, MET)                                                      \
  do {                                                                                 \
    constexpr int U = fused_u(MODE);                                                   \
    auto kern = k_fused_local<MODE, MASK, MET, U>;                                     \
    int grid = stream_grid(kern, kBlock, ntiles, (kBlock / 32) * U);                   \
    launch_pdl(kern, grid, kBlock, 0, st, theta, m, g, mask, n, h, hp->lr, hp->weight_decay, \
                                  fill, sq, sign_bits, nz_bits, tie_bits, flags);      \
  } while (0)
#define LC_FUSED_M(MODE)                         \
  do {                                           \
    if (mask) {                                  \
      if (metrics) LC_FUSED(MODE, true, true);   \
      else LC_FUSED(MODE, true, false);          \
    } else {                                     \
      if (metrics) LC_FUSED(MODE, false, true);  \
      else LC_FUSED(MODE, false, false);         \
    }                                            \
  } while (0)
  switch (mode) {
    case LC_LOCAL_BINARY: LC_FUSED_M(LC_LOCAL_BINARY); break;
    case LC_LOCAL_PS: LC_FUSED_M(LC_LOCAL_PS); break;
    case LC_LOCAL_QUANT:
      if (needs_quant_x(segs)) LC_FUSED_M(kLocalQuantX);
      else LC_FUSED_M(LC_LOCAL_QUANT);
      break;
    default: return set_err(LC_E_ARG, "lc_fused_local_step: unknown mode %d", mode);
  }
#undef LC_FUSED_M
#undef LC_FUSED
  LC_LAUNCH_CHECK();
  return LC_OK;
}

bool make_out(VoteOut& o, void* const* v, void* const* nz, void* const* tie, int nout) {
  const int nt = nout < 0 ? 1 : nout;  // nout == -1: one multicast address each
  if (nout < -1 || nout == 0 || !make_dst(o.v, v, nt)) return false;
  o.nout = nout;
  for (int i = 0; i < LC_MAX_BLOCKS; ++i) o.nz.p[i] = o.tie.p[i] = nullptr;
  if (nz && !make_dst(o.nz, nz, nt)) return false;
  if (tie && !make_dst(o.tie, tie, nt)) return false;
  return true;
}

int lc_vote_bits(const uint32_t* recv, int32_t P, int64_t cw, int64_t n_valid, int fill,
                 int sum_mode, void* const* voted, void* const* nz, void* const* tie_bits,
                 int32_t nout, uint32_t* flags, const lc_sync* sync, void* stream) {
  if (P < 1 || P > 255 || cw < 0 || (cw % 4) != 0 || !flags)
    return set_err(LC_E_ARG, "lc_vote_bits: P must be in [1,255], cw a multiple of 4");
  if (cw == 0) return sync_only(sync, stream);
  VoteOut o;
  if (!recv || !make_out(o, voted, nz, tie_bits, nout))
    return set_err(LC_E_ARG, "lc_vote_bits: bad pointers / output table");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int grid = generic_grid(cw / 4);
  const SyncD sy = to_syncd(sync);
#define LC_VOTE(NP) LC_CUDA_TRY(launch_pdl(k_vote_bits<NP>, grid, kBlock, 0, st, recv, P, cw, n_valid, fill, sum_mode, o, flags, sy))
  if (P <= 1) LC_VOTE(1);
  else if (P <= 3) LC_VOTE(2);
  else if (P <= 7) LC_VOTE(3);
  else if (P <= 15) LC_VOTE(4);
  else if (P <= 31) LC_VOTE(5);
  else if (P <= 63) LC_VOTE(6);
  else if (P <= 127) LC_VOTE(7);
  else LC_VOTE(8);
#undef LC_VOTE
  LC_LAUNCH_CHECK();
  return LC_OK;
}

namespace {
thread_local MeanArgs g_mean{};  // set by lc_vote_apply_sync for its launch (inline mode)
thread_local int g_va_cap = 0;   // > 0: k_vote_apply grid capped at this many CTAs per SM

// fork/join events of the side-stream mean, one pair per host thread
struct ForkEvents {
  cudaEvent_t fork = nullptr, join = nullptr;
  int dev = -1;
};
thread_local ForkEvents g_fork;

int fork_events(cudaEvent_t& fork, cudaEvent_t& join) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (g_fork.dev != dev) {
    if (g_fork.fork) cudaEventDestroy(g_fork.fork);
    if (g_fork.join) cudaEventDestroy(g_fork.join);
    LC_CUDA_TRY(cudaEventCreateWithFlags(&g_fork.fork, cudaEventDisableTiming));
    LC_CUDA_TRY(cudaEventCreateWithFlags(&g_fork.join, cudaEventDisableTiming));
    g_fork.dev = dev;
  }
  fork = g_fork.fork;
  join = g_fork.join;
  return LC_OK;
}
}  // namespace

// CTAs per SM of the vote/update grid and of the side-stream mean while they
// run together (LIONCUB_SYNC_SIDE_CTAS="va,mean" overrides).  The mean needs
// few SMs to saturate NVLink stores, the theta update wants HBM bandwidth;
// at P = 2 half of each mean element stays local, so the mean needs more.
// Measured, 7e9 params, whole sync step:
//   4 x B200: 3,1 69.7 ms; 2,1 67.8; 2,2 69.5; 4,1 73.7; 1,2 78.4
//             (serial kernels 75.0, the mean inside the vote grid 75.8)
//   2 x B200: 2,1 60.5 ms; 1,2 50.9; 2,2 50.2; 2,4 50.2; 1,6 57.9
//   after the vote/update redesign and the interleaved K1 (4 x B200):
//             2,1 65.5 ms; 2,2 65.3; 3,1 66.6; 1,1 66.4 (tests/sweep_side3.sh)
struct SideCtas {
  int va, mean;
};
SideCtas side_ctas(int P) {
  static const SideCtas env = [] {
    SideCtas v{0, 0};
    if (const char* e = std::getenv("LIONCUB_SYNC_SIDE_CTAS")) {
      int a = 0, b = 0;
      if (std::sscanf(e, "%d,%d", &a, &b) == 2 && a > 0 && b > 0) v = SideCtas{a, b};
    }
    return v;
  }();
  if (env.va > 0) return env;
  return P <= 2 ? SideCtas{2, 2} : SideCtas{2, 1};
}

int lc_vote_apply_sync(const uint32_t* recv, int32_t P, int64_t cw, int64_t n_valid, int fill,
                       int sum_mode, void* const* voted, void* const* nz, int32_t nout,
                       uint32_t* flags, const lc_sync* sync, float* theta, int64_t n,
                       const uint32_t* full, const uint32_t* nz_full, double lr, double wd,
                       const float* mean_stage, void* const* mean_out, int64_t mean_L,
                       int64_t mean_cnt, uint32_t* mean_work, void* side_stream, void* stream) {
  MeanArgs ma{};
  if (!mean_stage || !mean_out || !mean_work || mean_L <= 0 || (mean_L % 4) != 0 ||
      mean_cnt < 0 || mean_cnt > mean_L || !make_dst(ma.out, mean_out, P))
    return set_err(LC_E_ARG, "lc_vote_apply_sync: bad momentum-mean arguments");
  if ((reinterpret_cast<uintptr_t>(mean_stage) & 15u) != 0)
    return set_err(LC_E_ARG, "lc_vote_apply_sync: staging must be 16-byte aligned");
  for (int k = 0; k < P; ++k)
    if ((reinterpret_cast<uintptr_t>(ma.out.p[k]) & 15u) != 0)
      return set_err(LC_E_ARG, "lc_vote_apply_sync: momentum blocks must be 16-byte aligned");
  ma.stage = mean_cnt > 0 ? mean_stage : nullptr;
  ma.L = mean_L;
  ma.cnt = mean_cnt;
  ma.work = mean_work;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  LC_CUDA_TRY(cudaMemsetAsync(mean_work, 0, sizeof(uint32_t), st));
  if (!side_stream) {  // inline: every CTA joins the mean after its theta share
    g_mean = ma;
    const int rc = lc_vote_apply(recv, P, cw, n_valid, fill, sum_mode, voted, nz, nout, flags,
                                 sync, theta, n, full, nz_full, lr, wd, stream);
    g_mean = MeanArgs{};
    return rc;
  }
  // side stream: fork after K1 (and the work-counter reset), the lean mean
  // kernel fills the SMs the capped vote/update grid leaves free, join
  cudaStream_t side = reinterpret_cast<cudaStream_t>(side_stream);
  cudaEvent_t fork, join;
  if (int rc = fork_events(fork, join)) return rc;
  LC_CUDA_TRY(cudaEventRecord(fork, st));
  LC_CUDA_TRY(cudaStreamWaitEvent(side, fork, 0));
  g_va_cap = side_ctas(P).va;
  const int rc = lc_vote_apply(recv, P, cw, n_valid, fill, sum_mode, voted, nz, nout, flags, sync,
                               theta, n, full, nz_full, lr, wd, stream);
  g_va_cap = 0;
  if (rc) return rc;
  if (ma.stage) {
    SyncD wait = to_syncd(sync);
    wait.arrive_epoch = 0;  // the mean publishes nothing (the caller's barrier follows)
    int grid = stream_grid(k_sync_mean, kBlock, (mean_cnt + kMeanChunk - 1) / kMeanChunk, 1);
    if (grid > sm_count() * side_ctas(P).mean) grid = sm_count() * side_ctas(P).mean;
    LC_CUDA_TRY(launch_pdl(k_sync_mean, grid, kBlock, 0, side, wait, ma, (int)P));
    LC_LAUNCH_CHECK();
  }
  LC_CUDA_TRY(cudaEventRecord(join, side));
  LC_CUDA_TRY(cudaStreamWaitEvent(st, join, 0));
  return LC_OK;
}

int lc_set_vote_cap(int32_t ctas_per_sm) {
  if (ctas_per_sm < 0) return set_err(LC_E_ARG, "lc_set_vote_cap: ctas_per_sm >= 0");
  g_va_cap = ctas_per_sm;
  return LC_OK;
}

int lc_sync_mean(const lc_sync* wait, const float* stage, void* const* out, int32_t P, int64_t L,
                 int64_t cnt, uint32_t* work, int32_t ctas_per_sm, void* stream) {
  MeanArgs ma{};
  if (P < 1 || P > LC_MAX_BLOCKS || !stage || !work || L <= 0 || (L % 4) != 0 || cnt < 0 ||
      cnt > L || !make_dst(ma.out, out, P) || (reinterpret_cast<uintptr_t>(stage) & 15u))
    return set_err(LC_E_ARG, "lc_sync_mean: bad arguments");
  for (int k = 0; k < P; ++k)
    if ((reinterpret_cast<uintptr_t>(ma.out.p[k]) & 15u) != 0)
      return set_err(LC_E_ARG, "lc_sync_mean: outputs must be 16-byte aligned");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  LC_CUDA_TRY(cudaMemsetAsync(work, 0, sizeof(uint32_t), st));
  if (cnt == 0) return LC_OK;
  ma.stage = stage;
  ma.L = L;
  ma.cnt = cnt;
  ma.work = work;
  SyncD w = to_syncd(wait);
  w.arrive_epoch = 0;
  int grid = stream_grid(k_sync_mean, kBlock, (cnt + kMeanChunk - 1) / kMeanChunk, 1);
  if (ctas_per_sm > 0 && grid > sm_count() * ctas_per_sm) grid = sm_count() * ctas_per_sm;
  LC_CUDA_TRY(launch_pdl(k_sync_mean, grid, kBlock, 0, st, w, ma, (int)P));
  LC_LAUNCH_CHECK();
  return LC_OK;
}

int lc_vote_apply(const uint32_t* recv, int32_t P, int64_t cw, int64_t n_valid, int fill,
                  int sum_mode, void* const* voted, void* const* nz, int32_t nout,
                  uint32_t* flags, const lc_sync* sync, float* theta, int64_t n,
                  const uint32_t* full, const uint32_t* nz_full, double lr, double wd,
                  void* stream) {
  if (P < 1 || P > 32 || cw <= 0 || (cw % 4) != 0 || !flags || !sync || !sync->arrive_epoch)
    return set_err(LC_E_ARG, "lc_vote_apply: P in [1,32], cw % 4 == 0, sync with arrive_epoch");
  VoteOut o;
  if (!recv || !theta || !full || !make_out(o, voted, nz, nullptr, nout) || (nz && !nz_full))
    return set_err(LC_E_ARG, "lc_vote_apply: bad pointers / output table");
  if (!aligned16(theta)) return set_err(LC_E_ARG, "lc_vote_apply: theta must be 16-byte aligned");
  if ((int64_t)P * cw * 32 < n) return set_err(LC_E_ARG, "lc_vote_apply: blocks do not cover n");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const SyncD sy = to_syncd(sync);
  // work items of up to LC_VA_CHUNK super-tiles: large vectors keep the
  // counter's atomics few (one address: ~2.5 ns each), small ones keep the
  // items short (the last item is the tail)
  const int64_t nsup = (n + 1023) >> 10;
  const int64_t chunk = std::min<int64_t>(LC_VA_CHUNK, std::max<int64_t>(1, (nsup + LC_VA_ITEMS - 1) / LC_VA_ITEMS));
  ApplyArgs a{theta, n, full, nz_full, lr, wd, cw, chunk};
#define LC_VA(NP, NZ)                                                                      \
  do {                                                                                     \
    auto kern = g_mean.stage ? k_vote_apply<NP, NZ, true, false>                          \
                : g_va_cap > 0 ? k_vote_apply<NP, NZ, false, false>                       \
                               : k_vote_apply<NP, NZ, false, true>;                        \
    int grid = stream_grid(kern, kBlock, (n + 1023) >> 10, kBlock / 32);                   \
    if (g_va_cap > 0 && grid > sm_count() * g_va_cap) grid = sm_count() * g_va_cap;       \
    LC_CUDA_TRY(launch_pdl(kern, grid, kBlock, 0, st, recv, P, cw, n_valid, fill, sum_mode, \
                           o, flags, sy, a, g_mean));                                      \
  } while (0)
#define LC_VA_NZ(NP) do { if (nz) LC_VA(NP, true); else LC_VA(NP, false); } while (0)
  if (P <= 1) LC_VA_NZ(1);
  else if (P <= 3) LC_VA_NZ(2);
  else if (P <= 7) LC_VA_NZ(3);
  else if (P <= 15) LC_VA_NZ(4);
  else if (P <= 31) LC_VA_NZ(5);
  else LC_VA_NZ(6);
#undef LC_VA_NZ
#undef LC_VA
  LC_LAUNCH_CHECK();
  return LC_OK;
}

int lc_vote_update(const uint32_t* rows, int64_t row_stride, int32_t P, float* theta, int64_t n,
                   int fill, int sum_mode, double lr, double wd, uint32_t* flags,
                   const lc_sync* sync, void* stream) {
  if (n < 0 || P < 1 || P > 255 || !flags) return set_err(LC_E_ARG, "lc_vote_update: bad arguments");
  if (n == 0) return sync_only(sync, stream);
  if (!rows || !theta || row_stride < (n + 31) / 32)
    return set_err(LC_E_ARG, "lc_vote_update: null pointer / rows shorter than ceil(n/32)");
  if (!aligned16(theta)) return set_err(LC_E_ARG, "lc_vote_update: theta must be 16-byte aligned");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const SyncD sy = to_syncd(sync);
  const int64_t nsup = (n + 1023) >> 10;
#define LC_VU(NP, NZ)                                                                      \
  do {                                                                                     \
    auto kern = k_vote_update<NP, NZ>;                                                     \
    int grid = stream_grid(kern, kBlock, nsup, kBlock / 32);                               \
    LC_CUDA_TRY(launch_pdl(kern, grid, kBlock, 0, st, rows, row_stride, P, theta, n, fill, \
                           sum_mode, lr, wd, flags, sy));                                  \
  } while (0)
#define LC_VU_Z(NP) do { if (fill == 0) LC_VU(NP, true); else LC_VU(NP, false); } while (0)
  if (P <= 1) LC_VU_Z(1);
  else if (P <= 3) LC_VU_Z(2);
  else if (P <= 7) LC_VU_Z(3);
  else if (P <= 15) LC_VU_Z(4);
  else if (P <= 31) LC_VU_Z(5);
  else if (P <= 63) LC_VU_Z(6);
  else if (P <= 127) LC_VU_Z(7);
  else LC_VU_Z(8);
#undef LC_VU_Z
#undef LC_VU
  LC_LAUNCH_CHECK();
  return LC_OK;
}

int lc_fields_vote(const uint32_t* sums, int32_t rows, int64_t row_stride, int64_t n,
                   int32_t F, int32_t P, int32_t offset, int32_t binary, int fill,
                   void* const* voted, void* const* nz, void* const* tie_bits, int32_t nout,
                   int64_t* values, const lc_sync* sync, void* stream) {
  if (n < 0 || P < 1 || rows < 1) return set_err(LC_E_ARG, "lc_fields_vote: bad arguments");
  if (n == 0) return sync_only(sync, stream);
  VoteOut o;
  if (!sums || !make_out(o, voted, nz, tie_bits, nout))
    return set_err(LC_E_ARG, "lc_fields_vote: bad pointers / output table");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int64_t nin = (n * F + 31) / 32;
  int grid = generic_grid(nin);
  const SyncD sy = to_syncd(sync);
  if (!values && (row_stride % 4) == 0 && (reinterpret_cast<uintptr_t>(sums) & 15u) == 0) {
    const int gw = generic_grid((n + 31) / 32);
#define LC_FW(FF) LC_CUDA_TRY(launch_pdl(k_fields_vote_words<FF>, gw, kBlock, 0, st, sums, rows, row_stride, n, P, offset, binary, fill, o, sy))
    switch (F) {
      case 1: LC_FW(1); break;
      case 2: LC_FW(2); break;
      case 4: LC_FW(4); break;
      case 8: LC_FW(8); break;
      case 16: LC_FW(16); break;
      case 32: LC_FW(32); break;
      default: return set_err(LC_E_ARG, "lc_fields_vote: field_bits %d", F);
    }
#undef LC_FW
    LC_LAUNCH_CHECK();
    return LC_OK;
  }
#define LC_FV(FF) LC_CUDA_TRY(launch_pdl(k_fields_vote<FF>, grid, kBlock, 0, st, sums, rows, row_stride, n, P, offset, binary, fill, o, values, sy))
  switch (F) {
    case 1: LC_FV(1); break;
    case 2: LC_FV(2); break;
    case 4: LC_FV(4); break;
    case 8: LC_FV(8); break;
    case 16: LC_FV(16); break;
    case 32: LC_FV(32); break;
    default: return set_err(LC_E_ARG, "lc_fields_vote: field_bits %d", F);
  }
#undef LC_FV
  LC_LAUNCH_CHECK();
  return LC_OK;
}

int lc_f64_sum_vote(const double* recv, int32_t P, int64_t len, int64_t stride, int tree, int fill,
                    void* const* voted, void* const* nz, void* const* tie_bits, int32_t nout,
                    double* values, const lc_sync* sync, void* stream) {
  if (len < 0 || P < 1 || (tree && P > 64) || nout > 32)
    return set_err(LC_E_ARG, "lc_f64_sum_vote: bad arguments");
  if (len == 0) return sync_only(sync, stream);
  VoteOut o;
  if (!recv || !make_out(o, voted, nz, tie_bits, nout))
    return set_err(LC_E_ARG, "lc_f64_sum_vote: bad pointers / output table");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int grid = generic_grid(len);
  LC_CUDA_TRY(launch_pdl(k_f64_sum_vote, grid, kBlock, 0, st, recv, P, len, stride, tree, fill, o,
                         values, to_syncd(sync)));
  LC_LAUNCH_CHECK();
  return LC_OK;
}

int lc_mean_f32(const float* recv, int32_t P, int64_t len, int64_t stride, float* out,
                void* stream) {
  if (len < 0 || P < 1) return set_err(LC_E_ARG, "lc_mean_f32: bad arguments");
  if (len == 0) return LC_OK;
  if (!recv || !out) return set_err(LC_E_ARG, "lc_mean_f32: null pointer");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  k_mean_f32<<<generic_grid(len), kBlock, 0, st>>>(recv, P, len, stride, out);
  LC_LAUNCH_CHECK();
  return LC_OK;
}

int lc_compute_c(const float* g, const float* m, const uint8_t* mask, int64_t n,
                 const lc_hyper* hp, double* c, void* stream) {
  if (n < 0 || !hp) return set_err(LC_E_ARG, "lc_compute_c: bad arguments");
  if (n == 0) return LC_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  k_compute_c<<<generic_grid(n), kBlock, 0, st>>>(g, m, mask, n, to_hyp(hp), c);
  LC_LAUNCH_CHECK();
  return LC_OK;
}

int lc_count_bits_segmented(const uint32_t* bits, const int64_t* seg_start, int32_t nseg,
                            int64_t* counts, void* stream) {
  if (nseg < 1 || !bits || !seg_start || !counts)
    return set_err(LC_E_ARG, "lc_count_bits_segmented: bad arguments");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  LC_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(int64_t) * nseg, st));
  // total length lives on the device; size the grid generously
  k_count_bits_seg<<<sm_count() * 4, kBlock, 0, st>>>(bits, seg_start, nseg, counts);
  LC_LAUNCH_CHECK();
  return LC_OK;
}

int lc_bits_to_sign(const uint32_t* sign_bits, const uint32_t* nz_bits, int64_t n,
                    int8_t* out, void* stream) {
  if (n < 0) return set_err(LC_E_ARG, "lc_bits_to_sign: n < 0");
  if (n == 0) return LC_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  k_bits_to_sign<<<generic_grid(n), kBlock, 0, st>>>(sign_bits, nz_bits, n, out);
  LC_LAUNCH_CHECK();
  return LC_OK;
}

int lc_pack_i64_fields(const int64_t* v, int64_t n, int32_t F, int32_t offset,
                       int32_t binary, uint32_t* out, uint32_t* flags, void* stream) {
  if (n < 0 || !flags) return set_err(LC_E_ARG, "lc_pack_i64_fields: bad arguments");
  if (n == 0) return LC_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int grid = generic_grid((n * F + 31) / 32);
#define LC_PK(FF) k_pack_i64<FF><<<grid, kBlock, 0, st>>>(v, n, offset, binary, out, flags)
  switch (F) {
    case 1: LC_PK(1); break;
    case 2: LC_PK(2); break;
    case 4: LC_PK(4); break;
    case 8: LC_PK(8); break;
    case 16: LC_PK(16); break;
    case 32: LC_PK(32); break;
    default: return set_err(LC_E_ARG, "lc_pack_i64_fields: field_bits %d", F);
  }
#undef LC_PK
  LC_LAUNCH_CHECK();
  return LC_OK;
}

int lc_fields_decode(const uint32_t* sums, int64_t n, int32_t F, int32_t P, int32_t offset,
                     int32_t binary, int64_t* out, void* stream) {
  if (n < 0) return set_err(LC_E_ARG, "lc_fields_decode: n < 0");
  if (n == 0) return LC_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int grid = generic_grid(n);
#define LC_FD(FF) k_fields_decode<FF><<<grid, kBlock, 0, st>>>(sums, n, P, offset, binary, out)
  switch (F) {
    case 1: LC_FD(1); break;
    case 2: LC_FD(2); break;
    case 4: LC_FD(4); break;
    case 8: LC_FD(8); break;
    case 16: LC_FD(16); break;
    case 32: LC_FD(32); break;
    default: return set_err(LC_E_ARG, "lc_fields_decode: field_bits %d", F);
  }
#undef LC_FD
  LC_LAUNCH_CHECK();
  return LC_OK;
}

int lc_sign_pack_f64(const double* c, int64_t n, int fill, uint32_t* out, uint32_t* flags,
                     void* stream) {
  if (n < 0 || !flags) return set_err(LC_E_ARG, "lc_sign_pack_f64: bad arguments");
  if (n == 0) return LC_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  k_sign_pack_f64<<<generic_grid(n), kBlock, 0, st>>>(c, n, fill, out, flags);
  LC_LAUNCH_CHECK();
  return LC_OK;
}

int lc_sign_check(const float* g, const float* m, const uint8_t* mask, int64_t n,
                  const lc_hyper* hp, uint32_t* out, uint32_t* flags, void* stream) {
  if (n < 0 || !hp || !flags) return set_err(LC_E_ARG, "lc_sign_check: bad arguments");
  if (n == 0) return LC_OK;
  if (!g || !m) return set_err(LC_E_ARG, "lc_sign_check: null pointer");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  k_sign_check<<<generic_grid(n / 8), kBlock, 0, st>>>(g, m, mask, n, to_hyp(hp), out, flags);
  LC_LAUNCH_CHECK();
  return LC_OK;
}

int lc_sum_u32_rows(const uint32_t* const* rows, int32_t P, int64_t count, uint32_t* out,
                    void* stream) {
  if (P < 1 || P > 64 || count < 0 || !rows || !out)
    return set_err(LC_E_ARG, "lc_sum_u32_rows: bad arguments (P <= 64)");
  if (count == 0) return LC_OK;
  Rows r;
  for (int j = 0; j < P; ++j) r.p[j] = rows[j];
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  k_sum_rows<<<generic_grid(count), kBlock, 0, st>>>(r, P, count, out);
  LC_LAUNCH_CHECK();
  return LC_OK;
}

}  // extern "C"
