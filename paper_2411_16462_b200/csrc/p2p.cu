// NVLink peer-memory exchange for the Lion Cub step.
//
// With every rank's receive / gather buffers mapped into every other rank's
// address space (CUDA IPC for one process per GPU, peer access for one thread
// per GPU), the exchange needs no collective library: the encode kernel
// stores packed words straight into the owners' receive slots and the vote
// kernels store voted words into every rank's gather buffer.  What remains is
// ordering, provided by lc_barrier: a one-CTA kernel that publishes an epoch
// to every peer with a system-scope release store and waits (acquire loads,
// bounded by a timeout so a missing peer reports instead of hanging) until
// every peer has published the same epoch.
#include "common.cuh"

namespace {

struct Ptrs {
  void* p[LC_MAX_BLOCKS];
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void k_barrier(Ptrs peer_flags, uint64_t* __restrict__ my_flags, int P, int rank,
                          unsigned long long epoch, unsigned long long timeout_ns,
                          uint32_t* __restrict__ err) {
  const int j = threadIdx.x;
  if (j < P) {
    __threadfence_system();  // make this GPU's earlier peer stores visible first
    uint64_t* slot = reinterpret_cast<uint64_t*>(peer_flags.p[j]) + rank;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(slot), "l"(epoch) : "memory");
  }
  __syncthreads();
  if (j < P) {
    const unsigned long long t0 = globaltimer_ns();
    while (true) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(my_flags + j) : "memory");
      if (v >= epoch) break;
      if (globaltimer_ns() - t0 > timeout_ns) {
        atomicOr(err, (uint32_t)LC_FLAG_BARRIER_TIMEOUT);
        atomicOr(err + 1, 1u << (j & 31));  // the rank that never arrived
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
}

// dst[j][i] = src[j*s + i] for i < min(s, len - j*s): an owner-blocked
// scatter of one fp32 vector to P destinations (peer receive slots).  With
// src 16-byte aligned and s % 4 == 0 every quad stays inside one block and
// moves as one 128-bit load / (peer) store.
__global__ void __launch_bounds__(256)
k_push_blocks(const float* __restrict__ src, int64_t len, int64_t s, Ptrs dst, int P, int vec) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t done = 0;
  if (vec) {
    const int64_t nq = len >> 2;
    const float4* s4 = reinterpret_cast<const float4*>(src);
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += stride) {
      const int64_t e = q << 2;
      const int j = (int)(e / s);
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(dst.p[j]) + (e - (int64_t)j * s)) =
          __ldcs(s4 + q);
    }
    done = nq << 2;
  }
  for (int64_t e = done + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < len; e += stride) {
    const int j = (int)(e / s);
    reinterpret_cast<float*>(dst.p[j])[e - (int64_t)j * s] = __ldcs(src + e);
  }
}

__device__ __forceinline__ float mean_rows(const float* __restrict__ recv, int P, int64_t s,
                                           int64_t i, double dp) {
  double acc = (double)__ldcs(recv + i);
  for (int j = 1; j < P; ++j) acc = __dadd_rn(acc, (double)__ldcs(recv + (int64_t)j * s + i));
  return __double2float_rn(__ddiv_rn(acc, dp));
}

// out[k][i] = fp32( (sum_j f64(recv[j][i])) / P ) for every destination k:
// the reference's rank-ordered float64 mean (collectives.py:336-340), with
// the broadcast (:344) fused as peer stores, or as ONE NVLS multicast store
// (nout = -1).  Quads (128-bit rows/stores) when s and the outputs allow.
__global__ void __launch_bounds__(256)
k_mean_bcast(const float* __restrict__ recv, int P, int64_t cnt, int64_t s, Ptrs out, int nout,
             int vec) {
  const double dp = (double)P;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t done = 0;
  if (vec) {
    const int64_t nq = cnt >> 2;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += stride) {
      const int64_t i = q << 2;
      double acc[4];
      float4 x = __ldcs(reinterpret_cast<const float4*>(recv + i));
      acc[0] = x.x; acc[1] = x.y; acc[2] = x.z; acc[3] = x.w;
      for (int j = 1; j < P; ++j) {
        x = __ldcs(reinterpret_cast<const float4*>(recv + (int64_t)j * s + i));
        acc[0] = __dadd_rn(acc[0], (double)x.x);
        acc[1] = __dadd_rn(acc[1], (double)x.y);
        acc[2] = __dadd_rn(acc[2], (double)x.z);
        acc[3] = __dadd_rn(acc[3], (double)x.w);
      }
      float4 v;
      v.x = __double2float_rn(__ddiv_rn(acc[0], dp));
      v.y = __double2float_rn(__ddiv_rn(acc[1], dp));
      v.z = __double2float_rn(__ddiv_rn(acc[2], dp));
      v.w = __double2float_rn(__ddiv_rn(acc[3], dp));
      if (nout < 0) {
        asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};"
                     ::"l"(reinterpret_cast<float*>(out.p[0]) + i), "f"(v.x), "f"(v.y),
                     "f"(v.z), "f"(v.w) : "memory");
      } else {
        for (int k = 0; k < nout; ++k)
          *reinterpret_cast<float4*>(reinterpret_cast<float*>(out.p[k]) + i) = v;
      }
    }
    done = nq << 2;
  }
  for (int64_t i = done + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += stride) {
    const float v = mean_rows(recv, P, s, i, dp);
    if (nout < 0) {  // NVLS multicast: one store reaches every rank
      asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;"
                   ::"l"(reinterpret_cast<float*>(out.p[0]) + i), "f"(v) : "memory");
    } else {
      for (int k = 0; k < nout; ++k) reinterpret_cast<float*>(out.p[k])[i] = v;
    }
  }
}

// Owner-side momentum mean pulled straight from every rank's momentum over
// NVLink (no staging): element i of the owner's block, from P rows m_j[i],
// summed in float64 in rank order, divided once, rounded once to fp32, and
// stored to every rank (NVLS multicast, or one store per rank).
__global__ void __launch_bounds__(256)
k_mean_pull(Ptrs src, int P, int64_t off, int64_t cnt, Ptrs out, int nout, int vec,
            const uint32_t* __restrict__ err) {
  // the barrier before this kernel timed out: a peer's momentum is not final,
  // so nothing is averaged or stored (the step reports CollectiveError)
  if (err && (*reinterpret_cast<const volatile uint32_t*>(err) & LC_FLAG_BARRIER_TIMEOUT)) return;
  const double dp = (double)P;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t done = 0;
  if (vec) {
    const int64_t nq = cnt >> 2;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += stride) {
      const int64_t i = off + (q << 2);
      double acc[4];
      float4 x = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(src.p[0]) + i);
      acc[0] = x.x; acc[1] = x.y; acc[2] = x.z; acc[3] = x.w;
      for (int j = 1; j < P; ++j) {
        x = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(src.p[j]) + i);
        acc[0] = __dadd_rn(acc[0], (double)x.x);
        acc[1] = __dadd_rn(acc[1], (double)x.y);
        acc[2] = __dadd_rn(acc[2], (double)x.z);
        acc[3] = __dadd_rn(acc[3], (double)x.w);
      }
      float4 v;
      v.x = __double2float_rn(__ddiv_rn(acc[0], dp));
      v.y = __double2float_rn(__ddiv_rn(acc[1], dp));
      v.z = __double2float_rn(__ddiv_rn(acc[2], dp));
      v.w = __double2float_rn(__ddiv_rn(acc[3], dp));
      if (nout < 0) {
        asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};"
                     ::"l"(reinterpret_cast<float*>(out.p[0]) + i), "f"(v.x), "f"(v.y),
                     "f"(v.z), "f"(v.w) : "memory");
      } else {
        for (int k = 0; k < nout; ++k)
          *reinterpret_cast<float4*>(reinterpret_cast<float*>(out.p[k]) + i) = v;
      }
    }
    done = nq << 2;
  }
  for (int64_t t = done + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += stride) {
    const int64_t i = off + t;
    double acc = (double)__ldcv(reinterpret_cast<const float*>(src.p[0]) + i);
    for (int j = 1; j < P; ++j)
      acc = __dadd_rn(acc, (double)__ldcv(reinterpret_cast<const float*>(src.p[j]) + i));
    const float v = __double2float_rn(__ddiv_rn(acc, dp));
    if (nout < 0) {
      asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;"
                   ::"l"(reinterpret_cast<float*>(out.p[0]) + i), "f"(v) : "memory");
    } else {
      for (int k = 0; k < nout; ++k) reinterpret_cast<float*>(out.p[k])[i] = v;
    }
  }
}

bool make_ptrs(Ptrs& d, void* const* src, int n) {
  if (n < 1 || n > LC_MAX_BLOCKS || !src) return false;
  for (int i = 0; i < LC_MAX_BLOCKS; ++i) d.p[i] = i < n ? src[i] : nullptr;
  for (int i = 0; i < n; ++i)
    if (!d.p[i]) return false;
  return true;
}

int grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  int64_t cap = (int64_t)lc::sm_count() * 8;
  if (b > cap) b = cap;
  return b < 1 ? 1 : (int)b;
}

}  // namespace

extern "C" {

int lc_sym_alloc(int64_t bytes, void** ptr, uint8_t handle[64]) {
  if (bytes <= 0 || !ptr || !handle) return lc::set_err(LC_E_ARG, "lc_sym_alloc: bad arguments");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
  void* p = nullptr;
  LC_CUDA_TRY(cudaMalloc(&p, bytes));
  cudaError_t e = cudaMemset(p, 0, bytes);
  cudaIpcMemHandle_t h;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return lc::set_err(LC_E_CUDA, "lc_sym_alloc: %s", cudaGetErrorString(e));
  }
  memcpy(handle, &h, sizeof(h));
  *ptr = p;
  return LC_OK;
}

int lc_sym_free(void* ptr) {
  if (ptr) LC_CUDA_TRY(cudaFree(ptr));
  return LC_OK;
}

int lc_sym_open(const uint8_t handle[64], void** ptr) {
  if (!handle || !ptr) return lc::set_err(LC_E_ARG, "lc_sym_open: bad arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  LC_CUDA_TRY(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return LC_OK;
}

int lc_sym_close(void* ptr) {
  if (ptr) LC_CUDA_TRY(cudaIpcCloseMemHandle(ptr));
  return LC_OK;
}

int lc_enable_peer_access(int32_t device, int32_t peer) {
  int can = 0;
  LC_CUDA_TRY(cudaDeviceCanAccessPeer(&can, device, peer));
  if (!can) return lc::set_err(LC_E_CONFIG, "device %d cannot access peer %d", device, peer);
  int cur = 0;
  LC_CUDA_TRY(cudaGetDevice(&cur));
  LC_CUDA_TRY(cudaSetDevice(device));
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    e = cudaSuccess;
  }
  cudaSetDevice(cur);
  if (e != cudaSuccess) return lc::set_err(LC_E_CUDA, "peer access %d->%d: %s", device, peer, cudaGetErrorString(e));
  return LC_OK;
}

int lc_barrier(void* const* peer_flags, int32_t P, int32_t rank, uint64_t* my_flags,
               uint64_t epoch, double timeout_s, uint32_t* err, void* stream) {
  Ptrs pf;
  if (P < 1 || P > 32 || rank < 0 || rank >= P || !my_flags || !err || !make_ptrs(pf, peer_flags, P))
    return lc::set_err(LC_E_ARG, "lc_barrier: bad arguments");
  const unsigned long long ns = (unsigned long long)(timeout_s * 1e9);
  k_barrier<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(pf, my_flags, P, rank,
                                                                  epoch, ns, err);
  LC_LAUNCH_CHECK();
  return LC_OK;
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int lc_push_blocks_f32(const float* src, int64_t len, int64_t s, void* const* dst, int32_t P,
                       void* stream) {
  Ptrs d;
  if (len < 0 || s <= 0 || (len + s - 1) / s > P || !make_ptrs(d, dst, P))
    return lc::set_err(LC_E_ARG, "lc_push_blocks_f32: bad arguments");
  if (len == 0) return LC_OK;
  int vec = aligned16(src) && (s % 4) == 0;
  for (int j = 0; j < P && vec; ++j) vec = aligned16(d.p[j]);
  k_push_blocks<<<grid_for(vec ? len / 4 : len), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      src, len, s, d, P, vec);
  LC_LAUNCH_CHECK();
  return LC_OK;
}

int lc_mean_bcast_f32(const float* recv, int32_t P, int64_t cnt, int64_t s, void* const* out,
                      int32_t nout, void* stream) {
  Ptrs o;
  const int nt = nout < 0 ? 1 : nout;
  if (cnt < 0 || P < 1 || !recv || nout == 0 || nout < -1 || !make_ptrs(o, out, nt))
    return lc::set_err(LC_E_ARG, "lc_mean_bcast_f32: bad arguments");
  if (cnt == 0) return LC_OK;
  int vec = aligned16(recv) && (s % 4) == 0;
  for (int k = 0; k < nt && vec; ++k) vec = aligned16(o.p[k]);
  k_mean_bcast<<<grid_for(vec ? cnt / 4 : cnt), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      recv, P, cnt, s, o, nout, vec);
  LC_LAUNCH_CHECK();
  return LC_OK;
}

int lc_mean_pull_f32(void* const* src, int32_t P, int64_t off, int64_t cnt, void* const* out,
                     int32_t nout, const uint32_t* err, void* stream) {
  Ptrs sp, o;
  const int nt = nout < 0 ? 1 : nout;
  if (cnt < 0 || off < 0 || P < 1 || nout == 0 || nout < -1 || !make_ptrs(sp, src, P) ||
      !make_ptrs(o, out, nt))
    return lc::set_err(LC_E_ARG, "lc_mean_pull_f32: bad arguments");
  if (cnt == 0) return LC_OK;
  int vec = (off % 4) == 0;
  for (int j = 0; j < P && vec; ++j) vec = aligned16(sp.p[j]);
  for (int k = 0; k < nt && vec; ++k) vec = aligned16(o.p[k]);
  k_mean_pull<<<grid_for(vec ? cnt / 4 : cnt), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      sp, P, off, cnt, o, nout, vec, err);
  LC_LAUNCH_CHECK();
  return LC_OK;
}

}  // extern "C"
