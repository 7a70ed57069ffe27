// Collectives of one uneven ZeRO-3 DP group over NVLink peer memory.
//
// Every rank of a group exports one "arena" (CUDA IPC handle, mapped once by the
// other ranks, so every rank addresses every peer's buffers through NVSwitch):
// per parameter unit (a layer, the embedding, the head) a 16-byte flag record
// {param_ready, grad_ready, done_counter, pad} and the rank's persistent bf16
// parameter SHARD; plus the fp32 gradient window slots (full units, assigned
// identically on every rank of the group).  Gathered full parameters live in
// local window slots that peers never read.
//
// The two per-layer collectives the reference models (hetplan simulate.py:
// AllGather tasks :292-328 / :408-446, ReduceScatter :523-534, OptimStep
// :536-550) become:
//
//  * AllGather-v (zb_peer_allgather_v): wait until every peer published the
//    parameter shard of the previous step (param_ready >= epoch - 1), then pull
//    each rank's shard into [displ_p, displ_p + count_p) of a local full buffer
//    — with the copy engines (mode 0, no SMs taken from the concurrent GEMMs) or
//    with an SM kernel (mode 1, 16-byte loads, many requests in flight).
//  * ReduceScatter-v + scale + AdamW + bf16 cast, ONE kernel
//    (zb_peer_rs_adamw): publish grad_ready = epoch, wait for every peer's, then
//    for this rank's shard [lo, lo+n) sum the g fp32 gradient slices straight
//    out of the peers' grad buffers (NVLink loads), scale, apply AdamW to the
//    fp32 master / exp_avg / exp_avg_sq, and write the bf16 parameter shard in
//    place; the last CTA to finish publishes param_ready = epoch.  The reduced
//    gradient never round-trips through HBM.
//
// Ordering: a gradient window slot is handed to another unit only after
// zb_peer_wait saw every peer's param_ready of the slot's previous unit, which
// each peer publishes only after its fused kernel finished reading the slot.  A
// rank overwrites its parameter shard only in its fused kernel, which waits for
// every peer's grad_ready, published only after that peer's backward — hence
// after its last AllGather of the layer in the step.  Epochs are the
// device-resident step counter (CUDA-graph safe); flags are monotonic.
//
// All spins are bounded (default 120 s of %globaltimer, zb_peer_set_timeout; 0 =
// unbounded) and trap with a message instead of hanging.
#include "adam.cuh"
#include "zb_internal.h"

#include <cstdio>
#include <cstring>

namespace zb {

constexpr int kMaxPeers = 8;

struct PeerBases {
  char* base[kMaxPeers];
};

ZB_DEVICE uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

ZB_DEVICE uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

ZB_DEVICE void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

ZB_DEVICE void fence_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

static uint64_t g_timeout_ns = 120ull * 1000000000ull;

// Spin until (int)(*flag - target) >= 0.
ZB_DEVICE void wait_flag(const uint32_t* flag, uint32_t target, int who, int me,
                         uint64_t flag_off, uint64_t timeout_ns) {
  if ((int)(ld_acquire_sys(flag) - target) >= 0) return;
  const uint64_t t0 = global_ns();
  while ((int)(ld_acquire_sys(flag) - target) < 0) {
    __nanosleep(64);
    if (timeout_ns && global_ns() - t0 > timeout_ns) {
      printf("zorse peer: rank %d timeout waiting for peer %d flag@%llu >= %u (have %u)\n", me,
             who, (unsigned long long)flag_off, target, ld_acquire_sys(flag));
      __trap();
    }
  }
}

// Threads 0..g-1 of the block wait for peer t's flag; then the whole block proceeds.
ZB_DEVICE void block_wait_peers(const PeerBases& pb, int g, int me, uint64_t flag_off,
                                uint32_t target, uint64_t timeout_ns) {
  const int t = threadIdx.x;
  if (t < g && t != me)
    wait_flag(reinterpret_cast<const uint32_t*>(pb.base[t] + flag_off), target, t, me, flag_off,
              timeout_ns);
  if (t < g) fence_sys();
  __syncthreads();
}

// One CTA: optionally publish this rank's flag (at flag_off + publish_off) = epoch,
// then wait until every peer's flag at flag_off >= epoch + delta.  The waits of
// both collectives live in this single-CTA kernel, so a rank that runs ahead
// spins on one SM and never starves its own compute stream.
__global__ void peer_wait_kernel(PeerBases pb, int g, int me, uint64_t flag_off,
                                 const int* epoch, int delta, int publish, uint64_t timeout_ns) {
  const uint32_t e = (uint32_t)*epoch;
  if (publish && threadIdx.x == 0) {
    fence_sys();
    st_release_sys(reinterpret_cast<uint32_t*>(pb.base[me] + flag_off), e);
  }
  block_wait_peers(pb, g, me, flag_off, e + delta, timeout_ns);
}

__global__ void peer_signal_kernel(uint32_t* flag, const int* epoch, int delta) {
  fence_sys();
  st_release_sys(flag, (uint32_t)(*epoch + delta));
}

struct Segs {
  uint64_t src[kMaxPeers];  // byte offset of peer p's shard in its arena
  int64_t off[kMaxPeers];   // element offset of peer p's shard in the full buffer
  int64_t cnt[kMaxPeers];
};

// SM pull: every peer's shard copied into the local full buffer with 16-byte
// vectors (shards are 128-B aligned by the shard rule; the tail of the last one is
// done bytewise).
__global__ void __launch_bounds__(512) peer_pull_kernel(PeerBases pb, int g, int me, char* dst_base,
                                                         int elem_bytes, Segs segs) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  for (int p = 0; p < g; ++p) {
    const int64_t bytes = segs.cnt[p] * elem_bytes;
    const char* src = pb.base[p] + segs.src[p];
    char* dst = dst_base + segs.off[p] * elem_bytes;
    if (src == dst) continue;
    const int64_t n16 = bytes >> 4;
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    int64_t i = tid;
    for (; i + 3 * nth < n16; i += 4 * nth) {
      uint4 a = s4[i], b = s4[i + nth], c = s4[i + 2 * nth], d = s4[i + 3 * nth];
      d4[i] = a; d4[i + nth] = b; d4[i + 2 * nth] = c; d4[i + 3 * nth] = d;
    }
    for (; i < n16; i += nth) d4[i] = s4[i];
    for (int64_t j = (n16 << 4) + tid; j < bytes; j += nth) dst[j] = src[j];
  }
}

// Fused reduce-scatter-v + grad scale + AdamW + bf16 cast for this rank's shard.
// G = group size (template, so the per-peer loads stay in registers); each
// thread issues the G gradient loads (G-1 over NVLink) and the 3 state loads of
// U float4 groups before any arithmetic, to keep enough bytes in flight to
// cover the NVLink read latency.
template <int G, int U>
__global__ void __launch_bounds__(256) peer_rs_adamw_kernel(
    PeerBases pb, int me, uint64_t grad_off, int64_t lo, int64_t n, uint64_t flag_off,
    const int* epoch, float* __restrict__ master, float* __restrict__ exp_avg,
    float* __restrict__ exp_avg_sq, __nv_bfloat16* __restrict__ param, float* grad_out,
    float* sumsq, AdamParams a) {
  // grad_ready was published and every peer's awaited by the preceding
  // peer_wait_kernel on this stream.
  const uint32_t e = (uint32_t)(*epoch);
  uint32_t* my_flags = reinterpret_cast<uint32_t*>(pb.base[me] + flag_off);
  resolve_step(a);

  const float* src[G];
#pragma unroll
  for (int p = 0; p < G; ++p) src[p] = reinterpret_cast<const float*>(pb.base[p] + grad_off) + lo;

  float ss = 0.f;
  const int64_t n4 = n >> 2;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int64_t base = t0; base < n4; base += U * nth) {
    float4 acc[U][G], pm[U], m[U], v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * nth;
      if (i < n4) {
#pragma unroll
        for (int p = 0; p < G; ++p) acc[u][p] = reinterpret_cast<const float4*>(src[p])[i];
        pm[u] = reinterpret_cast<const float4*>(master)[i];
        m[u] = reinterpret_cast<const float4*>(exp_avg)[i];
        v[u] = reinterpret_cast<const float4*>(exp_avg_sq)[i];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * nth;
      if (i >= n4) break;
      float4 gs = acc[u][0];
#pragma unroll
      for (int p = 1; p < G; ++p) {
        gs.x += acc[u][p].x; gs.y += acc[u][p].y; gs.z += acc[u][p].z; gs.w += acc[u][p].w;
      }
      gs.x *= a.grad_scale; gs.y *= a.grad_scale; gs.z *= a.grad_scale; gs.w *= a.grad_scale;
      if (grad_out) reinterpret_cast<float4*>(grad_out)[i] = gs;
      ss += gs.x * gs.x + gs.y * gs.y + gs.z * gs.z + gs.w * gs.w;
      adam_elem(pm[u].x, m[u].x, v[u].x, gs.x, a);
      adam_elem(pm[u].y, m[u].y, v[u].y, gs.y, a);
      adam_elem(pm[u].z, m[u].z, v[u].z, gs.z, a);
      adam_elem(pm[u].w, m[u].w, v[u].w, gs.w, a);
      reinterpret_cast<float4*>(master)[i] = pm[u];
      reinterpret_cast<float4*>(exp_avg)[i] = m[u];
      reinterpret_cast<float4*>(exp_avg_sq)[i] = v[u];
      uint2 o;
      o.x = pack_bf16(pm[u].x, pm[u].y);
      o.y = pack_bf16(pm[u].z, pm[u].w);
      reinterpret_cast<uint2*>(param)[i] = o;
    }
  }
  for (int64_t i = (n4 << 2) + t0; i < n; i += nth) {
    float gsum = 0.f;
#pragma unroll
    for (int p = 0; p < G; ++p) gsum += src[p][i];
    gsum *= a.grad_scale;
    if (grad_out) grad_out[i] = gsum;
    float pmv = master[i], mv = exp_avg[i], vv = exp_avg_sq[i];
    ss += gsum * gsum;
    adam_elem(pmv, mv, vv, gsum, a);
    master[i] = pmv;
    exp_avg[i] = mv;
    exp_avg_sq[i] = vv;
    param[i] = __float2bfloat16(pmv);
  }
  __shared__ float red[8];
  if (sumsq) {
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x < 32) {
      float t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
      t = warp_sum(t);
      if (threadIdx.x == 0) atomicAdd(sumsq, t);
    }
  }
  // Last CTA out publishes the new parameter shard: per-CTA gpu-scope fence +
  // counter, then one system-scope fence and release store.
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t prev = atomicAdd(my_flags + 2, 1u);
    if (prev == gridDim.x - 1) {
      my_flags[2] = 0;
      fence_sys();
      st_release_sys(my_flags + 0, e);
    }
  }
}

template <int G>
static void launch_rs_adamw(int grid, cudaStream_t s, const PeerBases& pb, int me,
                            uint64_t grad_off, int64_t lo, int64_t n, uint64_t flag_off,
                            const int* epoch, float* master, float* m, float* v,
                            __nv_bfloat16* param, float* grad_out, float* sumsq,
                            const AdamParams& a) {
  peer_rs_adamw_kernel<G, 2><<<grid, 256, 0, s>>>(pb, me, grad_off, lo, n, flag_off, epoch,
                                                  master, m, v, param, grad_out, sumsq, a);
}

static int load_bases(PeerBases* pb, void* const* bases, int g, int me) {
  if (g < 1 || g > kMaxPeers) return set_error(ZB_ERR_INVALID, "peer: group size %d not in [1, 8]", g);
  if (me < 0 || me >= g) return set_error(ZB_ERR_INVALID, "peer: rank %d not in group of %d", me, g);
  std::memset(pb, 0, sizeof(*pb));
  for (int p = 0; p < g; ++p) {
    if (!bases[p]) return set_error(ZB_ERR_INVALID, "peer: base of rank %d is NULL", p);
    pb->base[p] = static_cast<char*>(bases[p]);
  }
  return 0;
}

typedef CUresult (*GetAddressRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);

}  // namespace zb

using namespace zb;

extern "C" int zb_peer_enable(int peer_device) {
  // Single-process multi-GPU use (tests / NVLink probes): map peer_device's memory
  // into the current device's address space.  Multi-process ranks use CUDA IPC.
  cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return 0;
  }
  return e == cudaSuccess ? 0 : set_cuda_error(e, "cudaDeviceEnablePeerAccess");
}

extern "C" int zb_peer_set_timeout(double seconds) {
  if (!(seconds >= 0.0)) return set_error(ZB_ERR_INVALID, "peer timeout must be >= 0");
  g_timeout_ns = (uint64_t)(seconds * 1e9);
  return 0;
}

extern "C" int zb_ipc_handle_size(void) { return (int)sizeof(cudaIpcMemHandle_t); }

extern "C" int zb_ipc_get_handle(const void* ptr, void* handle_out, uint64_t* offset_out) {
  static GetAddressRangeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return set_error(ZB_ERR_CUDA, "cuMemGetAddressRange unavailable");
    fn = reinterpret_cast<GetAddressRangeFn>(p);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  CUresult r = fn(&base, &size, (CUdeviceptr)ptr);
  if (r != CUDA_SUCCESS) return set_error(ZB_ERR_CUDA, "cuMemGetAddressRange failed (%d)", (int)r);
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, (void*)base);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaIpcGetMemHandle");
  std::memcpy(handle_out, &h, sizeof(h));
  *offset_out = (uint64_t)((CUdeviceptr)ptr - base);
  return 0;
}

extern "C" int zb_ipc_open(const void* handle, void** base_out) {
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(base_out, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? 0 : set_cuda_error(e, "cudaIpcOpenMemHandle");
}

extern "C" int zb_ipc_close(void* base) {
  cudaError_t e = cudaIpcCloseMemHandle(base);
  return e == cudaSuccess ? 0 : set_cuda_error(e, "cudaIpcCloseMemHandle");
}

extern "C" int zb_peer_signal(void* flag, const void* epoch_dev, int delta, cudaStream_t s) {
  peer_signal_kernel<<<1, 1, 0, s>>>((uint32_t*)flag, (const int*)epoch_dev, delta);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_cuda_error(e, "peer_signal");
}

extern "C" int zb_peer_wait(void* const* bases, int g, int me, uint64_t flag_off,
                            const void* epoch_dev, int epoch_delta, cudaStream_t s) {
  PeerBases pb;
  if (int rc = load_bases(&pb, bases, g, me)) return rc;
  if (!epoch_dev) return set_error(ZB_ERR_INVALID, "peer wait: NULL epoch");
  if (g == 1) return 0;
  peer_wait_kernel<<<1, 32, 0, s>>>(pb, g, me, flag_off, (const int*)epoch_dev, epoch_delta, 0,
                                       g_timeout_ns);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_cuda_error(e, "peer_wait");
}

extern "C" int zb_peer_allgather_v(void* const* bases, int g, int me, const uint64_t* shard_offs,
                                   void* dst, int elem_bytes, const int64_t* counts,
                                   const int64_t* displs, uint64_t flag_off,
                                   const void* epoch_dev, int epoch_delta, int mode,
                                   cudaStream_t s) {
  PeerBases pb;
  if (int rc = load_bases(&pb, bases, g, me)) return rc;
  if (!dst || !shard_offs || !counts || !displs || !epoch_dev)
    return set_error(ZB_ERR_INVALID, "peer allgather: NULL argument");
  Segs segs;
  std::memset(&segs, 0, sizeof(segs));
  for (int p = 0; p < g; ++p) {
    segs.src[p] = shard_offs[p];
    segs.off[p] = displs[p];
    segs.cnt[p] = counts[p];
    if (((displs[p] * elem_bytes) & 15) || (shard_offs[p] & 15) || ((uintptr_t)dst & 15))
      return set_error(ZB_ERR_INVALID, "peer allgather: segment %d not 16-byte aligned", p);
  }
  cudaError_t e;
  if (g > 1) {
    peer_wait_kernel<<<1, 32, 0, s>>>(pb, g, me, flag_off, (const int*)epoch_dev, epoch_delta, 0,
                                       g_timeout_ns);
    if ((e = cudaGetLastError()) != cudaSuccess) return set_cuda_error(e, "peer_wait");
  }
  char* d = static_cast<char*>(dst);
  if (mode == 0) {  // copy engines
    for (int p = 0; p < g; ++p) {
      const char* src = pb.base[p] + shard_offs[p];
      char* to = d + (size_t)displs[p] * elem_bytes;
      if (counts[p] == 0 || src == to) continue;
      e = cudaMemcpyAsync(to, src, (size_t)counts[p] * elem_bytes, cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) return set_cuda_error(e, "peer allgather copy");
    }
    return 0;
  }
  int64_t total = 0;
  for (int p = 0; p < g; ++p) total += counts[p] * elem_bytes;
  int64_t want = (total / 16 + 2047) / 2048;
  int grid = (int)(want < 1 ? 1 : (want > 64 ? 64 : want));
  peer_pull_kernel<<<grid, 512, 0, s>>>(pb, g, me, d, elem_bytes, segs);
  e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_cuda_error(e, "peer_pull");
}

extern "C" int zb_peer_rs_adamw(void* const* bases, int g, int me, uint64_t grad_off, int64_t lo,
                                int64_t n, uint64_t flag_off, const void* epoch_dev,
                                void* master, void* exp_avg, void* exp_avg_sq, void* param_bf16,
                                void* grad_out, void* sumsq, float lr, float beta1, float beta2,
                                float eps, float weight_decay, float grad_scale,
                                const void* step_dev, cudaStream_t s) {
  PeerBases pb;
  if (int rc = load_bases(&pb, bases, g, me)) return rc;
  if (!step_dev || !epoch_dev) return set_error(ZB_ERR_INVALID, "peer rs_adamw: NULL step/epoch");
  const uintptr_t al = (uintptr_t)master | (uintptr_t)exp_avg | (uintptr_t)exp_avg_sq |
                       (uintptr_t)grad_out | (uintptr_t)(grad_off + lo * 4);
  if ((al & 15) || ((uintptr_t)param_bf16 & 7))
    return set_error(ZB_ERR_INVALID, "peer rs_adamw: shard buffers must be 16-byte aligned");
  AdamParams a = make_adam_params(lr, beta1, beta2, eps, weight_decay, grad_scale, 0,
                                  (const int*)step_dev);
  int64_t want = (n / 4 + 511) / 512;   // 2 float4 per thread per pass
  int64_t cap = (int64_t)num_sms() * 2;  // ~100 registers: 2 CTAs of 256 per SM
  int grid = (int)(want < 1 ? 1 : (want < cap ? want : cap));
  const int* ep = (const int*)epoch_dev;
  float *pm = (float*)master, *m = (float*)exp_avg, *v = (float*)exp_avg_sq;
  __nv_bfloat16* pp = (__nv_bfloat16*)param_bf16;
  float *go = (float*)grad_out, *ss = (float*)sumsq;
  if (g > 1) {  // publish grad_ready = epoch, wait for every peer's
    peer_wait_kernel<<<1, 32, 0, s>>>(pb, g, me, flag_off + 4, ep, 0, 1, g_timeout_ns);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error(e, "peer_wait");
  }
  switch (g) {
#define ZB_RS_CASE(G_) \
    case G_: launch_rs_adamw<G_>(grid, s, pb, me, grad_off, lo, n, flag_off, ep, pm, m, v, pp, go, ss, a); break;
    ZB_RS_CASE(1) ZB_RS_CASE(2) ZB_RS_CASE(3) ZB_RS_CASE(4)
    ZB_RS_CASE(5) ZB_RS_CASE(6) ZB_RS_CASE(7) ZB_RS_CASE(8)
#undef ZB_RS_CASE
    default: return set_error(ZB_ERR_INVALID, "peer rs_adamw: group size %d", g);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_cuda_error(e, "peer_rs_adamw");
}
