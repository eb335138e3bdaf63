// peer.cu -- NVLink peer memory for the GWPS step on one NVSwitch box (a3, a8, a9 without NCCL kernels).
//
// Every rank exports its weight / gradient buffers with CUDA IPC once at init; peers map them and
//   - pull weight stripes with plain cudaMemcpyAsync on the weight stream: the copy engines move them over NVLink
//     while the persistent GEMM keeps all 148 SMs (the NCCL all-gather / P2P kernels of round 1 took SMs from it);
//   - read the group members' fp32 gradient stripes (and the other groups' rail partials) directly inside the fused
//     accumulate + AdamW kernel (kernels.cu: adamw_grouped) -- the reduce-scatter receive is that kernel's load.
// Ordering across processes uses monotone 32-bit sequence flags in each rank's signal array: a producer writes
// seq into the consumer's flag (a one-warp kernel: system-scope fence, then the peer store), the consumer's stream
// waits with cuStreamWaitValue32(flag >= seq), which the GPU front end polls without occupying an SM.
#include <cuda.h>
#include <nccl.h>

#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "peer.cuh"

namespace tp {

namespace {

using PFN_wait32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

PFN_wait32 get_wait32() {
  static PFN_wait32 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    TP_CUDA(cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q));
    TP_CHECK(q == cudaDriverEntryPointSuccess && p, TAWPIPE_ERUNTIME, "cuStreamWaitValue32 unavailable");
    fn = reinterpret_cast<PFN_wait32>(p);
  });
  return fn;
}

struct SigTargets {
  uint32_t* p[kMaxSignalTargets];
};

__global__ void signal_kernel(SigTargets t, int n, uint32_t value) {
  if (threadIdx.x < n) {
    __threadfence_system();   // everything this stream wrote or read before is ordered before the flag
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(t.p[threadIdx.x]), "r"(value) : "memory");
  }
}

// part[i] = W(Σ_members src_m[i]) in member order, fp32 (the non-owner group's reduce-scatter receive, a8)
template <typename W>
__global__ void __launch_bounds__(256) group_partial_kernel(PartialSources src, W* __restrict__ out, int64_t n) {
  const int64_t n4 = n / 4;
  for (int64_t i4 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i4 < n4;
       i4 += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    // peer memory: ld.global.cg, never through this SM's L1 (see kernels.cu ld8src)
    float4 acc = __ldcg(reinterpret_cast<const float4*>(src.p[0]) + i4);
    for (int m = 1; m < src.n; ++m) {
      const float4 x = __ldcg(reinterpret_cast<const float4*>(src.p[m]) + i4);
      acc.x += x.x;
      acc.y += x.y;
      acc.z += x.z;
      acc.w += x.w;
    }
    W* o = out + i4 * 4;
    o[0] = from_f<W>(acc.x);
    o[1] = from_f<W>(acc.y);
    o[2] = from_f<W>(acc.z);
    o[3] = from_f<W>(acc.w);
  }
}

}  // namespace

bool peer_open(ncclComm_t comm, int rank, int world, const std::vector<void*>& local,
               std::vector<std::vector<void*>>& remote, cudaStream_t s) {
  const int nb = static_cast<int>(local.size());
  constexpr int HS = sizeof(cudaIpcMemHandle_t);
  std::vector<char> mine(static_cast<size_t>(nb) * HS, 0);
  for (int b = 0; b < nb; ++b)
    if (local[b]) TP_CUDA(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(&mine[static_cast<size_t>(b) * HS]),
                                              local[b]));
  char* d_all = nullptr;
  const size_t per = static_cast<size_t>(nb) * HS;
  TP_CUDA(cudaMalloc(&d_all, per * world));
  TP_CUDA(cudaMemcpyAsync(d_all + per * rank, mine.data(), per, cudaMemcpyHostToDevice, s));
  ncclResult_t r = ncclAllGather(d_all + per * rank, d_all, per, ncclChar, comm, s);
  std::vector<char> all(per * world);
  if (r == ncclSuccess) {
    TP_CUDA(cudaMemcpyAsync(all.data(), d_all, per * world, cudaMemcpyDeviceToHost, s));
    TP_CUDA(cudaStreamSynchronize(s));
  }
  TP_CUDA(cudaFree(d_all));
  TP_CHECK(r == ncclSuccess, TAWPIPE_ERUNTIME, std::string("NCCL handle exchange: ") + ncclGetErrorString(r));
  remote.assign(world, std::vector<void*>(nb, nullptr));
  bool ok = true;
  for (int p = 0; p < world && ok; ++p) {
    for (int b = 0; b < nb; ++b) {
      if (p == rank) {
        remote[p][b] = local[b];
        continue;
      }
      cudaIpcMemHandle_t h;
      std::memcpy(&h, &all[per * p + static_cast<size_t>(b) * HS], HS);
      bool empty = true;
      for (int i = 0; i < HS; ++i) empty = empty && h.reserved[i] == 0;
      if (empty) continue;   // the peer has no such buffer
      void* ptr = nullptr;
      if (cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        ok = false;
        break;
      }
      remote[p][b] = ptr;
    }
  }
  // every rank must take the same decision (the caller falls back to NCCL everywhere otherwise)
  int* d_ok = nullptr;
  int h_ok = ok ? 1 : 0;
  TP_CUDA(cudaMalloc(&d_ok, sizeof(int)));
  TP_CUDA(cudaMemcpyAsync(d_ok, &h_ok, sizeof(int), cudaMemcpyHostToDevice, s));
  r = ncclAllReduce(d_ok, d_ok, 1, ncclInt, ncclMin, comm, s);
  TP_CUDA(cudaMemcpyAsync(&h_ok, d_ok, sizeof(int), cudaMemcpyDeviceToHost, s));
  TP_CUDA(cudaStreamSynchronize(s));
  TP_CUDA(cudaFree(d_ok));
  TP_CHECK(r == ncclSuccess, TAWPIPE_ERUNTIME, std::string("NCCL: ") + ncclGetErrorString(r));
  if (!h_ok) {
    peer_close(remote, rank);
    return false;
  }
  return true;
}

void peer_close(std::vector<std::vector<void*>>& remote, int rank) {
  for (int p = 0; p < static_cast<int>(remote.size()); ++p) {
    if (p == rank) continue;
    for (void* ptr : remote[p])
      if (ptr) cudaIpcCloseMemHandle(ptr);
  }
  remote.clear();
}

void signal_peers(uint32_t* const* flags, int n, uint32_t value, cudaStream_t s) {
  if (n <= 0) return;
  TP_CHECK(n <= kMaxSignalTargets, TAWPIPE_EINVARIANT, "signal_peers: too many targets");
  SigTargets t{};
  for (int i = 0; i < n; ++i) t.p[i] = flags[i];
  signal_kernel<<<1, 32, 0, s>>>(t, n, value);
  TP_CUDA(cudaGetLastError());
  g_kstats.launches++;
}

void wait_flag(const uint32_t* flag, uint32_t value, cudaStream_t s) {
  const CUresult r = get_wait32()(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(flag), value,
                                  CU_STREAM_WAIT_VALUE_GEQ);
  TP_CHECK(r == CUDA_SUCCESS, TAWPIPE_ERUNTIME, "cuStreamWaitValue32 failed: " + std::to_string(static_cast<int>(r)));
}

template <typename W>
void group_partial(const PartialSources& src, W* out, int64_t n, cudaStream_t s) {
  TP_CHECK(src.n >= 1 && src.n <= kMaxPartialSources && n % 4 == 0, TAWPIPE_ECONFIG,
           "group_partial: 1..8 sources, n % 4 == 0");
  int64_t blocks = (n / 4 + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  group_partial_kernel<W><<<static_cast<unsigned>(blocks < 1 ? 1 : blocks), 256, 0, s>>>(src, out, n);
  TP_CUDA(cudaGetLastError());
  g_kstats.launches++;
}
template void group_partial<float>(const PartialSources&, float*, int64_t, cudaStream_t);
template void group_partial<bf16>(const PartialSources&, bf16*, int64_t, cudaStream_t);

}  // namespace tp
