// Standalone quantizer operators of the drop-in quant API (quant.py):
// quantize's elementwise pass, dequantize, apply_sign and the f64 -> f32
// exactness check.  The per-layer norms come from l1norm.cu (lc_norm_scales);
// packing reuses lc_pack_i64_fields / lc_fields_decode (kernels.cu).
// All elementwise and HBM-streaming: grid-stride loops over a grid sized to
// the SM count.
#include "common.cuh"

namespace {

constexpr int kBlock = 256;

int grid_for(int64_t n) {
  int64_t b = (n + kBlock - 1) / kBlock;
  int64_t cap = (int64_t)lc::sm_count() * 8;
  if (b > cap) b = cap;
  return b < 1 ? 1 : (int)b;
}

// q = quantize(x) elementwise (quant.py:151-173) given the segment scales.
__global__ void k_quantize_values(const float* __restrict__ x, int64_t n, lc::SegQ sq,
                                  int64_t* __restrict__ q) {
  lc::SegCursorX cur;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    q[e] = lc::quant_x((double)x[e], sq, cur, e);
}

// y = q * mult; log map undone as sign(y) * s * expm1(|y|) (quant.py:183-195,
// :123-124), numpy's left-to-right order.
__global__ void k_dequantize(const int64_t* __restrict__ q, int64_t n, double mult,
                             double s, int log, double* __restrict__ out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double y = __dmul_rn((double)q[e], mult);
    if (!log) {
      out[e] = y;
    } else {
      const double sg = y > 0.0 ? 1.0 : (y < 0.0 ? -1.0 : 0.0);
      out[e] = __dmul_rn(__dmul_rn(sg, s), expm1(fabs(y)));
    }
  }
}

// apply_sign (quant.py:198-204): np.sign, zeros (incl. -0.0) -> fill.
template <typename T>
__global__ void k_apply_sign(const T* __restrict__ x, int64_t n, int fill,
                             int8_t* __restrict__ out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const T v = x[e];
    out[e] = v > T(0) ? 1 : (v < T(0) ? -1 : (v == T(0) ? (int8_t)fill : 0));
  }
}

__global__ void k_f64_to_f32_exact(const double* __restrict__ x, int64_t n,
                                   float* __restrict__ out, uint32_t* __restrict__ flags) {
  uint32_t bad = 0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[e];
    const float f = __double2float_rn(v);
    out[e] = f;
    if ((double)f != v && v == v) bad = 1;
  }
  if (bad) atomicOr(flags, (uint32_t)LC_FLAG_RANGE);
}

}  // namespace

extern "C" {

int lc_quantize_values(const float* x, int64_t n, const lc_segments* segs, int64_t* q,
                       void* stream) {
  if (n < 0 || !segs || !segs->start || !segs->scale || segs->nseg < 1)
    return lc::set_err(LC_E_ARG, "lc_quantize_values: bad arguments");
  if (n == 0) return LC_OK;
  if (!x || !q) return lc::set_err(LC_E_ARG, "lc_quantize_values: null pointer");
  lc::SegQ sq{segs->start, segs->scale, segs->nseg, segs->qmax, segs->log_scale,
              segs->qflags, segs->seed};
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  k_quantize_values<<<grid_for(n), kBlock, 0, st>>>(x, n, sq, q);
  LC_LAUNCH_CHECK();
  return LC_OK;
}

int lc_dequantize(const int64_t* q, int64_t n, double mult, double log_scale, int32_t log,
                  double* out, void* stream) {
  if (n < 0) return lc::set_err(LC_E_ARG, "lc_dequantize: n < 0");
  if (n == 0) return LC_OK;
  if (!q || !out) return lc::set_err(LC_E_ARG, "lc_dequantize: null pointer");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  k_dequantize<<<grid_for(n), kBlock, 0, st>>>(q, n, mult, log_scale, log, out);
  LC_LAUNCH_CHECK();
  return LC_OK;
}

int lc_apply_sign_values(const void* x, int32_t is_f64, int64_t n, int fill, int8_t* out,
                         void* stream) {
  if (n < 0 || fill < -1 || fill > 1) return lc::set_err(LC_E_ARG, "lc_apply_sign_values: bad arguments");
  if (n == 0) return LC_OK;
  if (!x || !out) return lc::set_err(LC_E_ARG, "lc_apply_sign_values: null pointer");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (is_f64)
    k_apply_sign<double><<<grid_for(n), kBlock, 0, st>>>(static_cast<const double*>(x), n, fill, out);
  else
    k_apply_sign<float><<<grid_for(n), kBlock, 0, st>>>(static_cast<const float*>(x), n, fill, out);
  LC_LAUNCH_CHECK();
  return LC_OK;
}

int lc_f64_to_f32_exact(const double* x, int64_t n, float* out, uint32_t* flags,
                        void* stream) {
  if (n < 0 || !flags) return lc::set_err(LC_E_ARG, "lc_f64_to_f32_exact: bad arguments");
  if (n == 0) return LC_OK;
  if (!x || !out) return lc::set_err(LC_E_ARG, "lc_f64_to_f32_exact: null pointer");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  k_f64_to_f32_exact<<<grid_for(n), kBlock, 0, st>>>(x, n, out, flags);
  LC_LAUNCH_CHECK();
  return LC_OK;
}

}  // extern "C"
