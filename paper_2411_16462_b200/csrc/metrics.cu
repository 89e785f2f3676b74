// Divergence metric of the reference (optimizer.py:261-276): per layer, the
// max over elements of the population std of momentum across ranks,
// np.stack(rows).std(axis=0, ddof=0).max().  numpy reduces axis 0 of a
// C-contiguous (P, n) array row by row, so the mean and the sum of squares
// are sequential in rank order (verified against np.std); every operation
// below is that order in float64, so the result is bit-identical.
#include <algorithm>

#include "common.cuh"

namespace {

constexpr int kBlock = 256;
constexpr int kTab = 64;  // per-CTA segment-max table

__global__ void __launch_bounds__(kBlock)
k_std_max(const float* __restrict__ rows, int P, int64_t n, int64_t stride,
          const int64_t* __restrict__ start, int nseg, int64_t per_cta,
          unsigned long long* __restrict__ out) {
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
  unsigned long long cur = 0ull;
  auto flush = [&]() {
    if (seg < 0 || !cur) return;
    if (use_tab) atomicMax(&tab[seg - s_first], cur);
    else atomicMax(&out[seg], cur);
  };
  const double inv_p = (double)P;
  for (int64_t e = lo + threadIdx.x; e < hi; e += blockDim.x) {
    if (e < seg_lo || e >= seg_hi) {
      flush();
      cur = 0ull;
      seg = lc::seg_find(start, nseg, e);
      seg_lo = start[seg];
      seg_hi = start[seg + 1];
    }
    double s = (double)__ldcs(rows + e);
    for (int r = 1; r < P; ++r) s = __dadd_rn(s, (double)__ldcs(rows + r * stride + e));
    const double mean = __ddiv_rn(s, inv_p);
    double v = 0.0;
    for (int r = 0; r < P; ++r) {
      const double d = __dsub_rn((double)rows[r * stride + e], mean);
      v = r == 0 ? __dmul_rn(d, d) : __dadd_rn(v, __dmul_rn(d, d));
    }
    const double sd = __dsqrt_rn(__ddiv_rn(v, inv_p));
    const unsigned long long b = (unsigned long long)__double_as_longlong(sd);
    cur = b > cur ? b : cur;
  }
  flush();
  __syncthreads();
  if (use_tab)
    for (int i = threadIdx.x; i <= s_last - s_first; i += blockDim.x)
      if (tab[i]) atomicMax(&out[s_first + i], tab[i]);
}

// runner.py:171-177: the vote sign against the sign of the full-precision
// aggregate ref = allreduce_mean_f32(c_local): match where equal and the vote
// is nonzero, flip where strictly opposite (both nonzero).  np.sign of a NaN
// mean is NaN, which matches nothing.
__global__ void __launch_bounds__(kBlock)
k_sign_agreement(const int8_t* __restrict__ vote, const float* __restrict__ ref, int64_t n,
                 unsigned long long* __restrict__ out) {
  unsigned long long match = 0, flip = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int v = vote[i];
    const float r = ref[i];
    const int s = r > 0.f ? 1 : (r < 0.f ? -1 : 0);
    const bool nan = r != r;
    match += (!nan && v != 0 && v == s);
    flip += (!nan && v != 0 && s != 0 && v == -s);
  }
  for (int o = 16; o; o >>= 1) {
    match += __shfl_xor_sync(0xffffffffu, match, o);
    flip += __shfl_xor_sync(0xffffffffu, flip, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(out, match);
    atomicAdd(out + 1, flip);
  }
}

}  // namespace

extern "C" {

int lc_sign_agreement(const int8_t* vote, const float* ref, int64_t n, int64_t* counts,
                      void* stream) {
  if (n < 0 || !counts) return lc::set_err(LC_E_ARG, "lc_sign_agreement: bad arguments");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  LC_CUDA_TRY(cudaMemsetAsync(counts, 0, 2 * sizeof(int64_t), st));
  if (n == 0) return LC_OK;
  if (!vote || !ref) return lc::set_err(LC_E_ARG, "lc_sign_agreement: null pointer");
  int64_t grid = (n + kBlock - 1) / kBlock;
  grid = std::min<int64_t>(grid, (int64_t)lc::sm_count() * 8);
  k_sign_agreement<<<(int)grid, kBlock, 0, st>>>(vote, ref, n,
                                                 reinterpret_cast<unsigned long long*>(counts));
  LC_LAUNCH_CHECK();
  return LC_OK;
}

int lc_std_max_segmented(const float* rows, int32_t P, int64_t n, int64_t stride,
                         const int64_t* seg_start, int32_t nseg, double* out_max,
                         void* stream) {
  if (P < 1 || n < 0 || stride < n || nseg < 1 || !seg_start || !out_max)
    return lc::set_err(LC_E_ARG, "lc_std_max_segmented: bad arguments");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  LC_CUDA_TRY(cudaMemsetAsync(out_max, 0, sizeof(double) * nseg, st));
  if (n == 0) return LC_OK;
  if (!rows) return lc::set_err(LC_E_ARG, "lc_std_max_segmented: null rows");
  const int64_t nct = (int64_t)lc::sm_count() * 8;
  const int64_t per = std::max<int64_t>((n + nct - 1) / nct, 1024);
  const int grid = (int)((n + per - 1) / per);
  k_std_max<<<grid, kBlock, 0, st>>>(rows, P, n, stride, seg_start, nseg, per,
                                     reinterpret_cast<unsigned long long*>(out_max));
  LC_LAUNCH_CHECK();
  return LC_OK;
}

}  // extern "C"
