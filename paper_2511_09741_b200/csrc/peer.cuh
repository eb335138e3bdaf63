// peer.cuh -- NVLink peer memory for the GWPS step (peer.cu): IPC mapping, sequence flags, group partial sums.
#pragma once
#include <nccl.h>

#include <cstdint>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace tp {

constexpr int kMaxSignalTargets = 32;
constexpr int kMaxPartialSources = 8;

// Export `local` (cudaMalloc base pointers, nullptr allowed) with CUDA IPC, all-gather the handles over `comm` and
// map every peer's buffers: remote[p][b] is rank p's buffer b in this process (remote[rank] = local).  COLLECTIVE.
// Returns false on every rank (nothing mapped) if any rank could not map a peer (no NVLink / P2P path).
bool peer_open(ncclComm_t comm, int rank, int world, const std::vector<void*>& local,
               std::vector<std::vector<void*>>& remote, cudaStream_t s);
void peer_close(std::vector<std::vector<void*>>& remote, int rank);

// On stream s, after everything before it: write `value` into each flag (peer-mapped uint32), system-scope release.
void signal_peers(uint32_t* const* flags, int n, uint32_t value, cudaStream_t s);
// Stream s waits until *flag >= value (front-end poll, no SM).
void wait_flag(const uint32_t* flag, uint32_t value, cudaStream_t s);

struct PartialSources {
  const float* p[kMaxPartialSources] = {};
  int n = 0;
};
// out[i] = W(Σ_m p[m][i]) summed in fp32 in member order; n % 4 == 0, 16-byte aligned
template <typename W>
void group_partial(const PartialSources& src, W* out, int64_t n, cudaStream_t s);

}  // namespace tp
