// numpy-exact per-layer L1 mean norm for the p-bit Lion Cub path.
//
// quant.py:81-104 computes M1 = max|c| * mean(|c|/max|c|).  np.mean sums
// float64 with numpy's pairwise algorithm: blocks of <= 128 elements use 8
// strided accumulators combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a
// sequential tail; larger blocks split at n/2 rounded down to a multiple of 8
// (checked against np.sum in tests/test_oracle.py).  The summation tree
// depends only on the layer length, so the plan precomputes it once:
//   * the tree is cut into CTA work items of <= kItem elements;
//   * every distinct work-item size gets a template (its <=128-element leaves
//     and the level-ordered internal additions);
//   * the additions above the work items run level by level in one CTA per
//     layer.
// Every addition happens in exactly numpy's order, so the norm and therefore
// the quantized integers are bit-identical to the reference.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <functional>
#include <map>
#include <vector>

#include <map>
#include <mutex>

#include "common.cuh"

namespace {

constexpr int64_t kItem = 8192;  // elements per work-item CTA
constexpr int kLeaf = 128;       // numpy PW_BLOCKSIZE
constexpr int kThreads = 256;

struct Op {
  int dst, left, right, height;
};

struct Tmpl {
  std::vector<int> leaf_rel, leaf_size;
  std::vector<Op> ops;  // sorted by height
  std::vector<int> lvl; // op index where each height starts (+ end)
  int root = 0;         // slot of the root
  int nslots = 0;
};

int64_t split_left(int64_t n) {
  int64_t n2 = n / 2;
  return n2 - (n2 % 8);
}

// Build a work-item template: leaves are slots [0, L), internals [L, ...).
void build_tmpl(int64_t size, Tmpl& t) {
  struct Node {
    bool leaf;
    int idx;
    int height;
  };
  std::vector<Op> raw;  // internal ops with provisional internal indices
  int nleaf = 0, nint = 0;
  std::vector<int> lrel, lsize;
  // recursive lambda
  std::function<Node(int64_t, int64_t)> rec = [&](int64_t off, int64_t n) -> Node {
    if (n <= kLeaf) {
      lrel.push_back((int)off);
      lsize.push_back((int)n);
      return Node{true, nleaf++, 0};
    }
    int64_t n2 = split_left(n);
    Node a = rec(off, n2);
    Node b = rec(off + n2, n - n2);
    Op op;
    op.dst = nint++;
    op.left = a.leaf ? a.idx : -(a.idx + 1);
    op.right = b.leaf ? b.idx : -(b.idx + 1);
    op.height = 1 + std::max(a.height, b.height);
    raw.push_back(op);
    return Node{false, op.dst, op.height};
  };
  Node root = rec(0, size);
  t.leaf_rel = lrel;
  t.leaf_size = lsize;
  auto slot = [&](int v) { return v >= 0 ? v : nleaf + (-v - 1); };
  t.ops.clear();
  for (auto& o : raw) t.ops.push_back(Op{nleaf + o.dst, slot(o.left), slot(o.right), o.height});
  std::stable_sort(t.ops.begin(), t.ops.end(),
                   [](const Op& a, const Op& b) { return a.height < b.height; });
  t.lvl.clear();
  int h = 0;
  for (size_t i = 0; i < t.ops.size(); ++i) {
    while (h < t.ops[i].height) {
      t.lvl.push_back((int)i);
      ++h;
    }
  }
  t.lvl.push_back((int)t.ops.size());
  t.root = root.leaf ? root.idx : nleaf + root.idx;
  t.nslots = nleaf + nint;
}

struct DevTmpl {
  int leaf_begin, nleaf, op_begin, nlvl, lvl_begin, root, nslots, pad;
};

struct DevSeg {
  int64_t start, n;
  int op_begin, nlvl, lvl_begin, root;
  int node_begin, node_count;  // the segment's tree nodes are contiguous
};

// k_l1_upper stages a segment's nodes in shared memory when they fit
constexpr int kUpperSmemNodes = 24576;  // 192 KB of doubles

}  // namespace

struct lc_l1_plan_s {
  int nseg = 0;
  int max_seg_nodes = 0;  // largest per-segment node count (k_l1_upper smem)
  int64_t n_total = 0;
  int n_items = 0, n_nodes = 0, max_slots = 0;
  std::vector<int64_t> seg_start;
  // device
  int64_t* d_seg_start = nullptr;
  DevSeg* d_seg = nullptr;
  DevTmpl* d_tmpl = nullptr;
  int* d_leaf_rel = nullptr;
  int* d_leaf_size = nullptr;
  int4* d_tops = nullptr;     // template ops (dst, left, right, -)
  int* d_tlvl = nullptr;      // template level starts
  int4* d_uops = nullptr;     // upper ops
  int* d_ulvl = nullptr;      // upper level starts
  int64_t* d_wi_off = nullptr;  // work-item absolute element offset
  int* d_wi_meta = nullptr;     // (seg, tmpl, node) triples
  int* d_wi_leaf0 = nullptr;    // first global leaf of each work item
  int64_t n_leaves = 0;
  int64_t* d_lf_start = nullptr;  // global leaves: absolute element offset
  uint32_t* d_lf_meta = nullptr;  // size (8 bits) | segment << 8
  double* d_lf_sum = nullptr;     // leaf sums
  double* d_nodes = nullptr;
  unsigned long long* d_max = nullptr;
};

namespace {

using lc::Hyp;

// Norm orders (lc_norm_scales): the per-element term of numpy's mean and the
// final root (quant.py:94-104).
enum { PK_1 = 0, PK_2 = 1, PK_HALF = 2, PK_GEN = 3, PK_0 = 4, PK_INF = 5 };

// |y| for y = c, or the log map y = sign(c) log1p(|c|/s) when s > 0
// (quant.py:119-120, :143-146): |y| = log1p(|c|/s).
template <bool LOG>
__device__ __forceinline__ double abs_y(double c, double s) {
  double a = fabs(c);
  if (LOG && s > 0.0) a = log1p(__ddiv_rn(a, s));
  return a;
}

// Per-segment max|y| as uint64 bit patterns (non-negative doubles order as
// unsigned integers), or with COUNT the number of nonzero |y| (p = 0).
// Each CTA walks a contiguous, 16-byte aligned element range (so it meets
// few segments) with 128-bit loads, 4 quads per thread in flight; per-lane
// results are merged in shared memory first.
template <bool LOG, bool COUNT>
__global__ void __launch_bounds__(kThreads)
k_l1_max(const float* __restrict__ g, const float* __restrict__ m,
         const uint8_t* __restrict__ mask, const int64_t* __restrict__ start,
         int nseg, int64_t n, int64_t per_cta, Hyp h, const double* __restrict__ logs,
         unsigned long long* __restrict__ gmax) {
  constexpr int kTab = 256;
  constexpr int QU = 4;
  __shared__ unsigned long long tab[kTab];
  const int64_t lo = (int64_t)blockIdx.x * per_cta;
  if (lo >= n) return;
  const int64_t hi = min(n, lo + per_cta);
  const int s_first = lc::seg_find(start, nseg, lo);
  const int s_last = lc::seg_find(start, nseg, hi - 1);
  const bool use_tab = (s_last - s_first) < kTab;
  for (int i = threadIdx.x; i < kTab; i += blockDim.x) tab[i] = 0ull;
  __syncthreads();
  int seg = -1;
  int64_t seg_lo = 1, seg_hi = 0;
  double sv = 0.0;  // log scale of the current segment
  unsigned long long cur = 0ull;
  auto bits = [](double x) { return (unsigned long long)__double_as_longlong(x); };
  auto acc = [&](double a) {
    if (COUNT) {
      cur += a > 0.0 ? 1ull : 0ull;
    } else {
      const unsigned long long b = bits(a);
      cur = b > cur ? b : cur;
    }
  };
  auto flush = [&]() {
    if (seg < 0 || !cur) return;
    if (use_tab) {
      if (COUNT) atomicAdd(&tab[seg - s_first], cur);
      else atomicMax(&tab[seg - s_first], cur);
    } else {
      if (COUNT) atomicAdd(&gmax[seg], cur);
      else atomicMax(&gmax[seg], cur);
    }
  };
  auto take = [&](int64_t e, float gv, float mv) {
    if (e < seg_lo || e >= seg_hi) {
      flush();
      cur = 0ull;
      seg = lc::seg_find(start, nseg, e);
      seg_lo = start[seg];
      seg_hi = start[seg + 1];
      if (LOG) sv = logs[seg];
    }
    double c = lc::lion_c(mv, gv, h);
    if (mask && !mask[e]) c = 0.0;
    acc(abs_y<LOG>(c, sv));
  };
  const float4* g4 = reinterpret_cast<const float4*>(g);
  const float4* m4 = reinterpret_cast<const float4*>(m);
  const int64_t q_lo = lo >> 2, q_hi = hi >> 2;  // full quads of this range
  for (int64_t q0 = q_lo + threadIdx.x; q0 < q_hi; q0 += (int64_t)QU * blockDim.x) {
    float4 gv[QU], mv[QU];
#pragma unroll
    for (int u = 0; u < QU; ++u) {
      const int64_t q = q0 + (int64_t)u * blockDim.x;
      if (q < q_hi) {
        gv[u] = __ldcs(g4 + q);
        mv[u] = __ldcs(m4 + q);
      }
    }
#pragma unroll
    for (int u = 0; u < QU; ++u) {
      const int64_t q = q0 + (int64_t)u * blockDim.x;
      if (q >= q_hi) continue;
      const int64_t e = 4 * q;
      if (!mask && e >= seg_lo && e + 4 <= seg_hi) {
        // the whole quad lies in the current segment: no per-element checks
        const double c0 = abs_y<LOG>(lc::lion_c(mv[u].x, gv[u].x, h), sv);
        const double c1 = abs_y<LOG>(lc::lion_c(mv[u].y, gv[u].y, h), sv);
        const double c2 = abs_y<LOG>(lc::lion_c(mv[u].z, gv[u].z, h), sv);
        const double c3 = abs_y<LOG>(lc::lion_c(mv[u].w, gv[u].w, h), sv);
        if (COUNT) {
          acc(c0); acc(c1); acc(c2); acc(c3);
        } else {
          // max on the bit patterns (a NaN propagates like numpy's max)
          const unsigned long long b = max(max(bits(c0), bits(c1)), max(bits(c2), bits(c3)));
          cur = b > cur ? b : cur;
        }
      } else {
        take(e, gv[u].x, mv[u].x);
        take(e + 1, gv[u].y, mv[u].y);
        take(e + 2, gv[u].z, mv[u].z);
        take(e + 3, gv[u].w, mv[u].w);
      }
    }
  }
  for (int64_t e = (q_hi << 2) + threadIdx.x; e < hi; e += blockDim.x) take(e, g[e], m[e]);
  flush();
  __syncthreads();
  if (use_tab)
    for (int i = threadIdx.x; i <= s_last - s_first; i += blockDim.x)
      if (tab[i]) {
        if (COUNT) atomicAdd(&gmax[s_first + i], tab[i]);
        else atomicMax(&gmax[s_first + i], tab[i]);
      }
}

// a / b correctly rounded given y = RN(1/b): q = RN(a*y) is within one ulp
// of a/b, the FMA residual a - b*q is exact, and one correction q + r*y
// rounds to RN(a/b) (Markstein).  Valid for 0 <= a <= b with b normal and a
// normal result; the (rare) subnormal results take __ddiv_rn.
__device__ __forceinline__ double div_by(double a, double b, double y) {
  const double q = __dmul_rn(a, y);
  const double r = __fma_rn(-q, b, a);
  const double q2 = __fma_rn(r, y, q);
  if (q2 < 2.2250738585072014e-308 && a != 0.0) return __ddiv_rn(a, b);
  return q2;
}

struct Recip {
  double b, y;
  bool fast;
  __device__ __forceinline__ double operator()(double a) const {
    return fast ? div_by(a, b, y) : __ddiv_rn(a, b);
  }
};

__device__ __forceinline__ Recip make_recip(double mx) {
  Recip r;
  r.b = mx;
  r.y = __drcp_rn(mx);
  r.fast = mx >= 1e-300 && mx < 1e300;
  return r;
}

// The summed term of segment order PK for |y| = a: (a/max)**p with numpy's
// fast paths for p = 1 (copy), 2 (square), 0.5 (sqrt), else pow; p = 0:
// log(a) of the nonzero entries (zeros add +0.0, which leaves a sum as is).
template <int PK>
__device__ __forceinline__ double term(double a, const Recip& dv, double p) {
  if (PK == PK_0) return a > 0.0 ? log(a) : 0.0;
  const double t = dv(a);
  if (PK == PK_1) return t;
  if (PK == PK_2) return __dmul_rn(t, t);
  if (PK == PK_HALF) return __dsqrt_rn(t);
  return pow(t, p);
}

template <bool MASK, int PK, bool LOG>
__device__ __forceinline__ double l1_v(const float* g, const float* m, const uint8_t* mask,
                                       int64_t e, const Hyp& h, const Recip& dv, double sv,
                                       double p) {
  double c = lc::lion_c(m[e], g[e], h);
  if (MASK && !mask[e]) c = 0.0;
  return term<PK>(abs_y<LOG>(c, sv), dv, p);
}

// One CTA per work item: leaves with 8 lanes each, then templated additions.
#ifndef LC_L1_ITEM_THREADS
#define LC_L1_ITEM_THREADS 256
#endif
constexpr int kItemThreads = LC_L1_ITEM_THREADS;

template <bool MASK, int PK, bool LOG>
__global__ void __launch_bounds__(kItemThreads, 1024 / kItemThreads)
k_l1_items(const float* __restrict__ g, const float* __restrict__ m,
           const uint8_t* __restrict__ mask, Hyp h,
           const unsigned long long* __restrict__ gmax, const double* __restrict__ logs,
           double p, const int64_t* __restrict__ wi_off, const int* __restrict__ wi_meta,
           const DevTmpl* __restrict__ tmpl, const int* __restrict__ leaf_rel,
           const int* __restrict__ leaf_size, const int4* __restrict__ tops,
           const int* __restrict__ tlvl, double* __restrict__ nodes) {
  extern __shared__ double slots[];
  const int item = blockIdx.x;
  const int64_t base = wi_off[item];
  const int seg = wi_meta[3 * item], ti = wi_meta[3 * item + 1], node = wi_meta[3 * item + 2];
  const DevTmpl T = tmpl[ti];
  // max|y| (or, for p = 0, the nonzero count: only its being 0 matters here)
  const double mx = PK == PK_0 ? (double)gmax[seg] : __longlong_as_double((long long)gmax[seg]);
  if (mx == 0.0) {  // lp_mean_norm returns 0 before summing (quant.py:101-103)
    if (threadIdx.x == 0) nodes[node] = 0.0;
    return;
  }
  const double sv = LOG ? logs[seg] : 0.0;
  const Recip dv = make_recip(PK == PK_0 ? 1.0 : mx);
  const int lane = threadIdx.x & 31;
  const int k = lane & 7;
  const int group = threadIdx.x >> 3;
  const int ngroups = blockDim.x >> 3;
  for (int lf = group; lf < T.nleaf; lf += ngroups) {
    const int rel = leaf_rel[T.leaf_begin + lf];
    const int sz = leaf_size[T.leaf_begin + lf];
    const int64_t e0 = base + rel;
    const unsigned gm = 0xffu << (lane & 24);  // the 8 lanes of this leaf
    double res;
    if (sz < 8) {  // only a whole tiny layer: sequential from 0
      res = 0.0;
      if (k == 0)
        for (int i = 0; i < sz; ++i)
          res = __dadd_rn(res, l1_v<MASK, PK, LOG>(g, m, mask, e0 + i, h, dv, sv, p));
    } else {
      // lane k owns accumulator r_k over elements k, k+8, ... of the leaf's
      // full 8-groups (<= 16 of them): issue every load first, then add in
      // numpy's order
      const int ngrp = sz >> 3;
      float gv[16], mv[16];
      uint32_t keep = 0xffffu;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (i < ngrp) {
          gv[i] = __ldcs(g + e0 + 8 * i + k);
          mv[i] = __ldcs(m + e0 + 8 * i + k);
          if (MASK && !mask[e0 + 8 * i + k]) keep &= ~(1u << i);
        }
      }
      double r = 0.0;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (i < ngrp) {
          double c = lc::lion_c(mv[i], gv[i], h);
          if (MASK && !((keep >> i) & 1u)) c = 0.0;
          const double v = term<PK>(abs_y<LOG>(c, sv), dv, p);
          r = i == 0 ? v : __dadd_rn(r, v);
        }
      }
      // ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)); IEEE addition is commutative
      r = __dadd_rn(r, __shfl_xor_sync(gm, r, 1));
      r = __dadd_rn(r, __shfl_xor_sync(gm, r, 2));
      r = __dadd_rn(r, __shfl_xor_sync(gm, r, 4));
      res = r;
      if (k == 0)
        for (int i = ngrp * 8; i < sz; ++i)
          res = __dadd_rn(res, l1_v<MASK, PK, LOG>(g, m, mask, e0 + i, h, dv, sv, p));
    }
    if (k == 0) slots[lf] = res;
  }
  __syncthreads();
  for (int lv = 0; lv < T.nlvl; ++lv) {
    const int b = tlvl[T.lvl_begin + lv], e = tlvl[T.lvl_begin + lv + 1];
    for (int o = b + threadIdx.x; o < e; o += blockDim.x) {
      const int4 op = tops[T.op_begin + o];
      slots[op.x] = __dadd_rn(slots[op.y], slots[op.z]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) nodes[node] = slots[T.root];
}

// ---------------------------------------------------------------------------
// Leaf-parallel pipeline: every numpy leaf (<= 128 elements, 8 strided
// accumulators) of every layer is summed by an 8-lane group in one flat
// grid-stride pass (no per-item trees, all 16 loads per lane in flight), then
// one warp per work item combines its leaves with the item's template tree.
// ---------------------------------------------------------------------------
// (a/max)**p etc. of |y| = a; FAST divides by the reciprocal y = RN(1/max)
// with one Markstein correction, which is RN(a/max) whenever the quotient
// is normal (validated bitwise by lc_debug_div_check); else IEEE __ddiv_rn.
// Why FAST needs no per-element guard: c = RN(RN(b1 m) + RN((1-b1) g)) of
// fp32 m, g is a multiple of 2^-202 (each rounded product of an fp32 value
// >= 2^-149 with a double has ulp >= 2^-202), so a nonzero a >= 2^-202 and
// a/max is normal whenever max < 2^819 (k_l1_leaves checks the range; the
// log map, whose a can be tiny, always takes IEEE division).
template <int PK, bool FAST>
__device__ __forceinline__ double term_div(double a, double b, double y, double p) {
  if (PK == PK_0) return a > 0.0 ? log(a) : 0.0;
  double t;
  if (FAST) {
    const double q = __dmul_rn(a, y);
    t = __fma_rn(__fma_rn(-q, b, a), y, q);
  } else {
    t = __ddiv_rn(a, b);
  }
  if (PK == PK_1) return t;
  if (PK == PK_2) return __dmul_rn(t, t);
  if (PK == PK_HALF) return __dsqrt_rn(t);
  return pow(t, p);
}

// Sum of one numpy leaf (group of 8 lanes, lane k = accumulator k).
template <bool MASK, int PK, bool LOG, bool FAST>
__device__ __forceinline__ double leaf_sum(const float* __restrict__ g, const float* __restrict__ m,
                                           const uint8_t* __restrict__ mask, const Hyp& h,
                                           int64_t e0, int sz, int k, unsigned gm, double b,
                                           double y, double sv, double p) {
  auto one = [&](int64_t e) {
    double c = lc::lion_c(m[e], g[e], h);
    if (MASK && !mask[e]) c = 0.0;
    return term_div<PK, FAST>(abs_y<LOG>(c, sv), b, y, p);
  };
  double res = 0.0;
  if (sz < 8) {  // only a whole tiny layer: sequential from 0
    if (k == 0)
      for (int i = 0; i < sz; ++i) res = __dadd_rn(res, one(e0 + i));
    return res;
  }
  // one predicated group per step: the compiler keeps the loads of several
  // groups in flight (measured faster than staging all 32 loads in
  // registers first, which spills at 64 registers)
  const int ngrp = sz >> 3;
  double r = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if (i < ngrp) {
      const int64_t e = e0 + 8 * i + k;
      double c = lc::lion_c(__ldcs(m + e), __ldcs(g + e), h);
      if (MASK && !mask[e]) c = 0.0;
      const double v = term_div<PK, FAST>(abs_y<LOG>(c, sv), b, y, p);
      r = i == 0 ? v : __dadd_rn(r, v);
    }
  }
  r = __dadd_rn(r, __shfl_xor_sync(gm, r, 1));
  r = __dadd_rn(r, __shfl_xor_sync(gm, r, 2));
  r = __dadd_rn(r, __shfl_xor_sync(gm, r, 4));
  res = r;
  if (k == 0)
    for (int i = ngrp * 8; i < sz; ++i) res = __dadd_rn(res, one(e0 + i));
  return res;
}

// The rare general case (log map, extreme max) out of line, so the IEEE
// division does not weigh on the fast path's registers.
template <bool MASK, int PK, bool LOG>
__device__ __noinline__ double leaf_sum_ieee(const float* __restrict__ g,
                                             const float* __restrict__ m,
                                             const uint8_t* __restrict__ mask, Hyp h, int64_t e0,
                                             int sz, int k, unsigned gm, double b, double sv,
                                             double p) {
  return leaf_sum<MASK, PK, LOG, false>(g, m, mask, h, e0, sz, k, gm, b, 0.0, sv, p);
}

#ifndef LC_L1_LEAF_MINB
#define LC_L1_LEAF_MINB 5  // 48 registers: 5 CTAs/SM (measured 0.451 -> 0.433 ms at GPT-2 size)
#endif
template <bool MASK, int PK, bool LOG>
__global__ void __launch_bounds__(kThreads, LC_L1_LEAF_MINB)
k_l1_leaves(const float* __restrict__ g, const float* __restrict__ m,
            const uint8_t* __restrict__ mask, Hyp h,
            const unsigned long long* __restrict__ gmax, const double* __restrict__ logs,
            double p, int64_t n_leaves, const int64_t* __restrict__ lf_start,
            const uint32_t* __restrict__ lf_meta, double* __restrict__ lf_sum) {
  const int lane = threadIdx.x & 31;
  const int k = lane & 7;
  const unsigned gm = 0xffu << (lane & 24);
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) >> 3;
  for (int64_t lf = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3; lf < n_leaves;
       lf += ngroups) {
    const int64_t e0 = __ldg(lf_start + lf);
    const uint32_t meta = __ldg(lf_meta + lf);
    const int sz = (int)(meta & 0xffu);
    const int seg = (int)(meta >> 8);
    const double mx = PK == PK_0 ? (double)gmax[seg] : __longlong_as_double((long long)gmax[seg]);
    if (mx == 0.0) {  // the tree writes 0 for this segment; nothing to sum
      if (k == 0) lf_sum[lf] = 0.0;
      continue;
    }
    const double sv = LOG ? logs[seg] : 0.0;
    // reciprocal division unless max is extreme or the log map is on
    // (term_div); p = 0 divides nothing
    const bool fast = PK == PK_0 || (!LOG && mx >= 0x1p-1000 && mx < 0x1p819);
    double res;
    if (fast)
      res = leaf_sum<MASK, PK, LOG, true>(g, m, mask, h, e0, sz, k, gm, mx,
                                          PK == PK_0 ? 0.0 : __drcp_rn(mx), sv, p);
    else
      res = leaf_sum_ieee<MASK, PK, LOG>(g, m, mask, h, e0, sz, k, gm, mx, sv, p);
    if (k == 0) lf_sum[lf] = res;
  }
}

// One warp per work item: its leaf sums -> the item's template tree (numpy's
// additions above the leaves) -> the item's node.  Slots live in shared
// memory, one region per warp; levels are ordered by __syncwarp.
constexpr int kTreeWarps = 8;
__global__ void __launch_bounds__(kTreeWarps * 32)
k_l1_item_trees(int n_items, const unsigned long long* __restrict__ gmax, int pk,
                const int* __restrict__ wi_meta, const int* __restrict__ wi_leaf0,
                const DevTmpl* __restrict__ tmpl, const int4* __restrict__ tops,
                const int* __restrict__ tlvl, const double* __restrict__ lf_sum,
                int max_slots, double* __restrict__ nodes) {
  extern __shared__ double tslots[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * kTreeWarps + w;
  if (item >= n_items) return;
  double* slots = tslots + (size_t)w * max_slots;
  const int seg = wi_meta[3 * item], ti = wi_meta[3 * item + 1], node = wi_meta[3 * item + 2];
  const DevTmpl T = tmpl[ti];
  const double mx = pk == PK_0 ? (double)gmax[seg] : __longlong_as_double((long long)gmax[seg]);
  if (mx == 0.0) {
    if (lane == 0) nodes[node] = 0.0;
    return;
  }
  const int l0 = wi_leaf0[item];
  for (int lf = lane; lf < T.nleaf; lf += 32) slots[lf] = lf_sum[l0 + lf];
  __syncwarp();
  for (int lv = 0; lv < T.nlvl; ++lv) {
    const int b = tlvl[T.lvl_begin + lv], e = tlvl[T.lvl_begin + lv + 1];
    for (int o = b + lane; o < e; o += 32) {
      const int4 op = tops[T.op_begin + o];
      slots[op.x] = __dadd_rn(slots[op.y], slots[op.z]);
    }
    __syncwarp();
  }
  if (lane == 0) nodes[node] = slots[T.root];
}

__global__ void k_div_check(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                            unsigned long long* __restrict__ bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const Recip dv = make_recip(b[i]);
    const double x = fabs(a[i]) <= b[i] ? fabs(a[i]) : b[i];
    if (__double_as_longlong(dv(x)) != __double_as_longlong(__ddiv_rn(x, b[i])))
      atomicAdd(bad, 1ull);
  }
}

__device__ __forceinline__ double seg_mx(const unsigned long long* gmax, int s, int pk) {
  return pk == PK_0 ? (double)gmax[s] : __longlong_as_double((long long)gmax[s]);
}

// One CTA per layer: the additions above the work items (level by level),
// then M_p and the quantizer scale (quant.py:94-104, :148-161).
__global__ void __launch_bounds__(kThreads)
k_l1_upper(const DevSeg* __restrict__ segs, const int4* __restrict__ uops,
           const int* __restrict__ ulvl, const unsigned long long* __restrict__ gmax,
           double* __restrict__ nodes, int pk, double p, int qmax,
           double* __restrict__ norms, double* __restrict__ scales) {
  extern __shared__ double snode[];
  const int s = blockIdx.x;
  const DevSeg S = segs[s];
  const double mx = seg_mx(gmax, s, pk);
  double root = 0.0;
  if (mx != 0.0 && pk != PK_INF) {
    if (S.node_count <= kUpperSmemNodes) {
      // the levels run in shared memory: one load of the item nodes, then
      // __syncthreads-separated levels without a global round trip each
      const int nb = S.node_begin;
      for (int i = threadIdx.x; i < S.node_count; i += blockDim.x) snode[i] = nodes[nb + i];
      __syncthreads();
      for (int lv = 0; lv < S.nlvl; ++lv) {
        const int b = ulvl[S.lvl_begin + lv], e = ulvl[S.lvl_begin + lv + 1];
        for (int o = b + threadIdx.x; o < e; o += blockDim.x) {
          const int4 op = uops[S.op_begin + o];
          snode[op.x - nb] = __dadd_rn(snode[op.y - nb], snode[op.z - nb]);
        }
        __syncthreads();
      }
      root = snode[S.root - nb];
    } else {
      for (int lv = 0; lv < S.nlvl; ++lv) {
        const int b = ulvl[S.lvl_begin + lv], e = ulvl[S.lvl_begin + lv + 1];
        for (int o = b + threadIdx.x; o < e; o += blockDim.x) {
          const int4 op = uops[S.op_begin + o];
          nodes[op.x] = __dadd_rn(nodes[op.y], nodes[op.z]);
        }
        __syncthreads();
      }
      root = nodes[S.root];
    }
  }
  if (threadIdx.x == 0) {
    double M = 0.0;
    if (mx != 0.0) {
      if (pk == PK_INF) {
        M = mx;                                                  // max|y|
      } else if (pk == PK_0) {
        M = exp(__ddiv_rn(root, mx));                            // exp(mean(log nz))
      } else {
        const double mean = __ddiv_rn(root, (double)S.n);        // np.mean
        double r = mean;                                         // mean ** (1/p)
        if (pk == PK_2) r = __dsqrt_rn(mean);
        else if (pk == PK_HALF) r = __dmul_rn(mean, mean);
        else if (pk == PK_GEN) r = pow(mean, __ddiv_rn(1.0, p));
        M = __dmul_rn(mx, r);
      }
    }
    norms[s] = M;
    scales[s] = (M == 0.0 || qmax == 0) ? 0.0
                : pk == PK_INF ? __ddiv_rn((double)qmax, M)
                               : __ddiv_rn((double)qmax, __dmul_rn(2.0, M));
  }
}

int norm_kind(double p) {
  if (p == 1.0) return PK_1;
  if (p == 2.0) return PK_2;
  if (p == 0.5) return PK_HALF;
  if (p == 0.0) return PK_0;
  if (std::isinf(p) && p > 0) return PK_INF;
  return PK_GEN;
}

// Plan tables live in stream-ordered allocations on a private non-blocking
// stream: creating or destroying a plan never synchronises the device (a
// cudaFree would wait for every stream -- including kernels of other ranks
// spinning on an in-kernel barrier for this thread's next launch).
cudaStream_t plan_stream() {
  static std::mutex mu;
  static std::map<int, cudaStream_t> streams;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = streams.find(dev);
  if (it != streams.end()) return it->second;
  cudaStream_t s = nullptr;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  streams.emplace(dev, s);
  return s;
}

template <typename T>
int dev_alloc(T** dst, size_t bytes) {
  LC_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(dst), bytes, plan_stream()));
  return LC_OK;
}

template <typename T>
int upload(T** dst, const std::vector<T>& v) {
  size_t bytes = std::max<size_t>(1, v.size()) * sizeof(T);
  LC_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(dst), bytes, plan_stream()));
  if (!v.empty())
    LC_CUDA_TRY(cudaMemcpyAsync(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice,
                                plan_stream()));
  // pageable source: wait for this copy only (the plan stream), not the device
  LC_CUDA_TRY(cudaStreamSynchronize(plan_stream()));
  return LC_OK;
}

void dev_free(void* p) {
  if (p) cudaFreeAsync(p, plan_stream());
}

}  // namespace

extern "C" {

int lc_l1_plan_destroy(lc_l1_plan_t p) {
  if (!p) return LC_OK;
  dev_free(p->d_seg_start);
  dev_free(p->d_seg);
  dev_free(p->d_tmpl);
  dev_free(p->d_leaf_rel);
  dev_free(p->d_leaf_size);
  dev_free(p->d_tops);
  dev_free(p->d_tlvl);
  dev_free(p->d_uops);
  dev_free(p->d_ulvl);
  dev_free(p->d_wi_off);
  dev_free(p->d_wi_meta);
  dev_free(p->d_wi_leaf0);
  dev_free(p->d_lf_start);
  dev_free(p->d_lf_meta);
  dev_free(p->d_lf_sum);
  dev_free(p->d_nodes);
  dev_free(p->d_max);
  delete p;
  return LC_OK;
}

int lc_l1_plan_create(lc_l1_plan_t* out, const int64_t* seg_start, int32_t nseg) {
  if (!out || !seg_start || nseg < 1) return lc::set_err(LC_E_ARG, "lc_l1_plan_create: bad arguments");
  for (int s = 0; s < nseg; ++s) {
    if (seg_start[s + 1] < seg_start[s]) return lc::set_err(LC_E_ARG, "segment offsets must be sorted");
    if (seg_start[s + 1] == seg_start[s])
      return lc::set_err(LC_E_CONFIG, "lp_mean_norm of an empty vector (segment %d)", s);
  }
  auto* p = new lc_l1_plan_s();
  p->nseg = nseg;
  p->seg_start.assign(seg_start, seg_start + nseg + 1);
  p->n_total = seg_start[nseg];

  std::map<int64_t, int> tmpl_of;
  std::vector<Tmpl> tmpls;
  std::vector<int64_t> wi_off;
  std::vector<int> wi_meta;
  std::vector<int4> uops;
  std::vector<int> ulvl;
  std::vector<DevSeg> dsegs;
  int node_ctr = 0;

  for (int s = 0; s < nseg; ++s) {
    const int64_t s0 = seg_start[s], n = seg_start[s + 1] - seg_start[s];
    std::vector<Op> ops;
    struct R {
      int node, height;
    };
    std::function<R(int64_t, int64_t)> rec = [&](int64_t off, int64_t len) -> R {
      if (len <= kItem) {
        auto it = tmpl_of.find(len);
        int ti;
        if (it == tmpl_of.end()) {
          Tmpl t;
          build_tmpl(len, t);
          ti = (int)tmpls.size();
          tmpls.push_back(std::move(t));
          tmpl_of[len] = ti;
        } else {
          ti = it->second;
        }
        int node = node_ctr++;
        wi_off.push_back(s0 + off);
        wi_meta.push_back(s);
        wi_meta.push_back(ti);
        wi_meta.push_back(node);
        return R{node, 0};
      }
      int64_t n2 = split_left(len);
      R a = rec(off, n2);
      R b = rec(off + n2, len - n2);
      int node = node_ctr++;
      int h = 1 + std::max(a.height, b.height);
      ops.push_back(Op{node, a.node, b.node, h});
      return R{node, h};
    };
    const int node_first = node_ctr;
    R root = rec(0, n);
    std::stable_sort(ops.begin(), ops.end(), [](const Op& a, const Op& b) { return a.height < b.height; });
    DevSeg ds;
    ds.start = s0;
    ds.n = n;
    ds.op_begin = (int)uops.size();
    ds.lvl_begin = (int)ulvl.size();
    ds.root = root.node;
    ds.node_begin = node_first;
    ds.node_count = node_ctr - node_first;
    int h = 0;
    for (size_t i = 0; i < ops.size(); ++i)
      while (h < ops[i].height) {
        ulvl.push_back((int)i);
        ++h;
      }
    ulvl.push_back((int)ops.size());
    ds.nlvl = h;
    for (auto& o : ops) uops.push_back(make_int4(o.dst, o.left, o.right, o.height));
    dsegs.push_back(ds);
  }

  std::vector<DevTmpl> dt;
  std::vector<int> leaf_rel, leaf_size, tlvl;
  std::vector<int4> tops;
  for (auto& t : tmpls) {
    DevTmpl d;
    d.leaf_begin = (int)leaf_rel.size();
    d.nleaf = (int)t.leaf_rel.size();
    d.op_begin = (int)tops.size();
    d.lvl_begin = (int)tlvl.size();
    d.nlvl = (int)t.lvl.size() - 1;
    d.root = t.root;
    d.nslots = t.nslots;
    d.pad = 0;
    leaf_rel.insert(leaf_rel.end(), t.leaf_rel.begin(), t.leaf_rel.end());
    leaf_size.insert(leaf_size.end(), t.leaf_size.begin(), t.leaf_size.end());
    for (auto& o : t.ops) tops.push_back(make_int4(o.dst, o.left, o.right, o.height));
    tlvl.insert(tlvl.end(), t.lvl.begin(), t.lvl.end());
    p->max_slots = std::max(p->max_slots, t.nslots);
    dt.push_back(d);
  }
  // global leaf list in item order (each item's leaves contiguous)
  std::vector<int> wi_leaf0;
  std::vector<int64_t> lf_start;
  std::vector<uint32_t> lf_meta;
  for (size_t it = 0; it < wi_off.size(); ++it) {
    const Tmpl& t = tmpls[wi_meta[3 * it + 1]];
    wi_leaf0.push_back((int)lf_start.size());
    for (size_t l = 0; l < t.leaf_rel.size(); ++l) {
      lf_start.push_back(wi_off[it] + t.leaf_rel[l]);
      lf_meta.push_back((uint32_t)t.leaf_size[l] | ((uint32_t)wi_meta[3 * it] << 8));
    }
  }
  if (nseg >= (1 << 24)) {
    delete p;
    return lc::set_err(LC_E_ARG, "lc_l1_plan_create: at most 2^24 segments");
  }
  p->n_leaves = (int64_t)lf_start.size();
  p->n_items = (int)wi_off.size();
  p->n_nodes = node_ctr;
  for (const DevSeg& d : dsegs) p->max_seg_nodes = std::max(p->max_seg_nodes, d.node_count);
  int rc = LC_OK;
  if ((rc = upload(&p->d_seg_start, p->seg_start)) ||
      (rc = upload(&p->d_seg, dsegs)) || (rc = upload(&p->d_tmpl, dt)) ||
      (rc = upload(&p->d_leaf_rel, leaf_rel)) || (rc = upload(&p->d_leaf_size, leaf_size)) ||
      (rc = upload(&p->d_tops, tops)) || (rc = upload(&p->d_tlvl, tlvl)) ||
      (rc = upload(&p->d_uops, uops)) || (rc = upload(&p->d_ulvl, ulvl)) ||
      (rc = upload(&p->d_wi_off, wi_off)) || (rc = upload(&p->d_wi_meta, wi_meta)) ||
      (rc = upload(&p->d_wi_leaf0, wi_leaf0)) || (rc = upload(&p->d_lf_start, lf_start)) ||
      (rc = upload(&p->d_lf_meta, lf_meta))) {
    lc_l1_plan_destroy(p);
    return rc;
  }
  if (dev_alloc(&p->d_nodes, sizeof(double) * std::max(1, p->n_nodes)) != LC_OK ||
      dev_alloc(&p->d_max, sizeof(unsigned long long) * nseg) != LC_OK ||
      dev_alloc(&p->d_lf_sum, sizeof(double) * std::max<int64_t>(1, p->n_leaves)) != LC_OK ||
      cudaStreamSynchronize(plan_stream()) != cudaSuccess) {
    lc_l1_plan_destroy(p);
    return lc::set_err(LC_E_CUDA, "lc_l1_plan_create: cudaMallocAsync failed");
  }
  *out = p;
  return LC_OK;
}

}  // extern "C"

namespace {

// LIONCUB_L1_ITEMS=1: the per-item CTA kernel (leaves + tree in one CTA)
// instead of the leaf-parallel pass + warp trees (A/B and cross-check).
const bool g_l1_items_legacy = [] {
  const char* e = std::getenv("LIONCUB_L1_ITEMS");
  return e && e[0] == '1';
}();

template <bool LOG, bool COUNT>
void launch_max(lc_l1_plan_t p, const float* g, const float* m, const uint8_t* mask, Hyp h,
                const double* logs, cudaStream_t st) {
  const int64_t n = p->n_total;
  int64_t nct = (int64_t)lc::sm_count() * 8;
  int64_t per = (n + nct - 1) / nct;
  per = std::max<int64_t>((per + 4095) / 4096 * 4096, 4096);  // 16-byte aligned ranges
  int grid = (int)((n + per - 1) / per);
  k_l1_max<LOG, COUNT><<<grid, kThreads, 0, st>>>(g, m, mask, p->d_seg_start, p->nseg, n, per,
                                                  h, logs, p->d_max);
}

template <bool MASK, int PK, bool LOG>
int launch_items(lc_l1_plan_t p, const float* g, const float* m, const uint8_t* mask, Hyp h,
                 const double* logs, double pv, cudaStream_t st) {
  size_t smem = sizeof(double) * std::max(1, p->max_slots);
  auto items = k_l1_items<MASK, PK, LOG>;
  if (smem > 48 * 1024)
    LC_CUDA_TRY(cudaFuncSetAttribute(items, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  items<<<p->n_items, kItemThreads, smem, st>>>(g, m, mask, h, p->d_max, logs, pv, p->d_wi_off,
                                            p->d_wi_meta, p->d_tmpl, p->d_leaf_rel,
                                            p->d_leaf_size, p->d_tops, p->d_tlvl, p->d_nodes);
  return LC_OK;
}

template <bool MASK, int PK, bool LOG>
int launch_leaves(lc_l1_plan_t p, const float* g, const float* m, const uint8_t* mask, Hyp h,
                  const double* logs, double pv, int pk, cudaStream_t st) {
  if (p->n_leaves > 0) {
    auto kern = k_l1_leaves<MASK, PK, LOG>;
    const int64_t groups_per_cta = kThreads / 8;
    int64_t grid = (p->n_leaves + groups_per_cta - 1) / groups_per_cta;
    grid = std::min<int64_t>(grid, (int64_t)lc::sm_count() * LC_L1_LEAF_MINB * 8);
    kern<<<(int)grid, kThreads, 0, st>>>(g, m, mask, h, p->d_max, logs, pv, p->n_leaves,
                                         p->d_lf_start, p->d_lf_meta, p->d_lf_sum);
    LC_LAUNCH_CHECK();
  }
  const size_t smem = sizeof(double) * std::max(1, p->max_slots) * kTreeWarps;
  if (smem > 48 * 1024)
    LC_CUDA_TRY(cudaFuncSetAttribute(k_l1_item_trees, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
  k_l1_item_trees<<<(p->n_items + kTreeWarps - 1) / kTreeWarps, kTreeWarps * 32, smem, st>>>(
      p->n_items, p->d_max, pk, p->d_wi_meta, p->d_wi_leaf0, p->d_tmpl, p->d_tops, p->d_tlvl,
      p->d_lf_sum, std::max(1, p->max_slots), p->d_nodes);
  return LC_OK;
}

template <int PK>
int items_pk(lc_l1_plan_t p, const float* g, const float* m, const uint8_t* mask, Hyp h,
             const double* logs, double pv, cudaStream_t st) {
  if (!g_l1_items_legacy) {
    if (mask)
      return logs ? launch_leaves<true, PK, true>(p, g, m, mask, h, logs, pv, PK, st)
                  : launch_leaves<true, PK, false>(p, g, m, mask, h, logs, pv, PK, st);
    return logs ? launch_leaves<false, PK, true>(p, g, m, mask, h, logs, pv, PK, st)
                : launch_leaves<false, PK, false>(p, g, m, mask, h, logs, pv, PK, st);
  }
  if (mask)
    return logs ? launch_items<true, PK, true>(p, g, m, mask, h, logs, pv, st)
                : launch_items<true, PK, false>(p, g, m, mask, h, logs, pv, st);
  return logs ? launch_items<false, PK, true>(p, g, m, mask, h, logs, pv, st)
              : launch_items<false, PK, false>(p, g, m, mask, h, logs, pv, st);
}

int norm_scales(lc_l1_plan_t p, const float* g, const float* m, const uint8_t* mask,
                const lc_hyper* hp, double pv, int qmax, const double* logs, double* norms,
                double* scales, cudaStream_t st) {
  Hyp h{hp->beta1, hp->one_minus_beta1, hp->beta2, hp->one_minus_beta2};
  const int pk = norm_kind(pv);
  LC_CUDA_TRY(cudaMemsetAsync(p->d_max, 0, sizeof(unsigned long long) * p->nseg, st));
  if (pk == PK_0) {
    if (logs) launch_max<true, true>(p, g, m, mask, h, logs, st);
    else launch_max<false, true>(p, g, m, mask, h, logs, st);
  } else {
    if (logs) launch_max<true, false>(p, g, m, mask, h, logs, st);
    else launch_max<false, false>(p, g, m, mask, h, logs, st);
  }
  LC_LAUNCH_CHECK();
  int rc = LC_OK;
  switch (pk) {
    case PK_1: rc = items_pk<PK_1>(p, g, m, mask, h, logs, pv, st); break;
    case PK_2: rc = items_pk<PK_2>(p, g, m, mask, h, logs, pv, st); break;
    case PK_HALF: rc = items_pk<PK_HALF>(p, g, m, mask, h, logs, pv, st); break;
    case PK_GEN: rc = items_pk<PK_GEN>(p, g, m, mask, h, logs, pv, st); break;
    case PK_0: rc = items_pk<PK_0>(p, g, m, mask, h, logs, pv, st); break;
    default: break;  // p = inf: the max is the norm
  }
  if (rc) return rc;
  LC_LAUNCH_CHECK();
  const size_t smem = sizeof(double) * (size_t)std::min(p->max_seg_nodes, kUpperSmemNodes);
  if (smem > 48 * 1024) {
    static bool attr_set[64] = {};  // the attribute is per kernel and device
    int dev = 0;
    LC_CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64 || !attr_set[dev]) {
      LC_CUDA_TRY(cudaFuncSetAttribute(k_l1_upper, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(sizeof(double) * kUpperSmemNodes)));
      if (dev >= 0 && dev < 64) attr_set[dev] = true;
    }
  }
  k_l1_upper<<<p->nseg, kThreads, smem, st>>>(p->d_seg, p->d_uops, p->d_ulvl, p->d_max,
                                              p->d_nodes, pk, pv, qmax, norms, scales);
  LC_LAUNCH_CHECK();
  return LC_OK;
}

}  // namespace

extern "C" {

int lc_l1_scales(lc_l1_plan_t p, const float* g, const float* m, const uint8_t* mask,
                 const lc_hyper* hp, int32_t qmax, double* norms, double* scales,
                 void* stream) {
  if (!p || !g || !m || !hp || !norms || !scales) return lc::set_err(LC_E_ARG, "lc_l1_scales: bad arguments");
  return norm_scales(p, g, m, mask, hp, 1.0, qmax, nullptr, norms, scales,
                     reinterpret_cast<cudaStream_t>(stream));
}

int lc_norm_scales(lc_l1_plan_t p, const float* g, const float* m, const uint8_t* mask,
                   const lc_hyper* hp, const lc_norm_spec* spec, double* norms,
                   double* scales, void* stream) {
  if (!p || !g || !m || !hp || !spec || !norms || !scales)
    return lc::set_err(LC_E_ARG, "lc_norm_scales: bad arguments");
  const double pv = spec->p;
  if (std::isnan(pv) || pv < 0) return lc::set_err(LC_E_CONFIG, "invalid norm order %g", pv);
  return norm_scales(p, g, m, mask, hp, pv, spec->qmax, spec->log_scale, norms, scales,
                     reinterpret_cast<cudaStream_t>(stream));
}

int lc_debug_div_check(const double* a, const double* b, int64_t n, uint64_t* mismatches,
                       void* stream) {
  if (n < 0 || !a || !b || !mismatches) return lc::set_err(LC_E_ARG, "lc_debug_div_check: bad arguments");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  LC_CUDA_TRY(cudaMemsetAsync(mismatches, 0, sizeof(uint64_t), st));
  if (n == 0) return LC_OK;
  k_div_check<<<lc::sm_count() * 8, 256, 0, st>>>(a, b, n, reinterpret_cast<unsigned long long*>(mismatches));
  LC_LAUNCH_CHECK();
  return LC_OK;
}

}  // extern "C"
