// Stable sorts of (64-bit key, 32-bit payload) pairs for the PauliSum
// engine's merges (PauliSum::from_terms over a batch of candidates,
// R:src/pauli.cpp:78-115): term products sorted by (segment, string) before
// the run sums. Keys compare on their low `end_bit` bits; equal keys keep
// their input order.
//
//   n <= kSmall   one CTA: bitonic network on (key, input position) in shared
//                 memory (one launch)
//   otherwise     LSD radix sort, 8-bit digits, ONE kernel per pass: the
//                 digit totals of every pass come from one histogram kernel
//                 up front; in a pass each CTA takes the next tile (a ticket
//                 counter, so every earlier tile is already resident), ranks
//                 its keys, publishes its per-digit count and finds its
//                 offset by looking back over the earlier tiles' published
//                 counts / inclusive prefixes (one 32-bit word carries flag
//                 and value), then scatters. A tile is 256 threads x 16
//                 items in memory order (warp-contiguous chunks, 32
//                 consecutive keys per round), ranks within a round from
//                 __match_any_sync, per-warp digit counters in shared memory.
//   n >= 2^30     the same ranking with a histogram kernel, a scan of the
//                 (digit, CTA) counts (scan.cuh) and a scatter per pass.
//
// The input is never written; the result lands in (kout, vout); `ws` holds
// workspace_bytes(n) bytes.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

#include "scan.cuh"

namespace liecl_b200 {
namespace sort {

using u64 = unsigned long long;

constexpr int kSmall = 2048;          // one-CTA limit
constexpr int kThreads = 256;         // radix CTA
constexpr int kItems = 16;            // keys per thread
constexpr int kTile = kThreads * kItems;
constexpr int kWarps = kThreads / 32;
constexpr int kBins = 256;

__device__ __forceinline__ u64 low_bits(u64 k, int bits) { return bits >= 64 ? k : (k & ((1ull << bits) - 1)); }

// ---- one CTA, n <= kSmall
__global__ void __launch_bounds__(1024) small_kernel(const u64* __restrict__ kin, const unsigned* __restrict__ vin,
                                                     int n, int end_bit, u64* __restrict__ kout,
                                                     unsigned* __restrict__ vout) {
  __shared__ u64 s_key[kSmall];   // masked key
  __shared__ unsigned s_pos[kSmall];
  int m = 1;
  while (m < n) m <<= 1;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    s_key[i] = i < n ? low_bits(kin[i], end_bit) : ~0ull;
    s_pos[i] = i < n ? static_cast<unsigned>(i) : 0xffffffffu;  // padding sorts last among equal keys
  }
  __syncthreads();
  for (int size = 2; size <= m; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < m / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));  // i with a zero inserted at the stride bit
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const u64 a = s_key[lo], b = s_key[hi];
        const unsigned pa = s_pos[lo], pb = s_pos[hi];
        const bool a_gt_b = a > b || (a == b && pa > pb);
        if (a_gt_b == up) {
          s_key[lo] = b, s_key[hi] = a;
          s_pos[lo] = pb, s_pos[hi] = pa;
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const unsigned p = s_pos[i];
    kout[i] = kin[p];
    vout[i] = vin[p];
  }
}

// ---- radix passes
// item `it` of thread (warp, lane) in tile `tile`: memory order
__device__ __forceinline__ int64_t item_index(int64_t tile, int warp, int lane, int it) {
  return tile * kTile + warp * (32 * kItems) + it * 32 + lane;
}

__global__ void __launch_bounds__(kThreads) hist_kernel(const u64* __restrict__ key, int64_t n, int shift, int bits,
                                                        int nblocks, int* __restrict__ counts) {
  __shared__ int s_hist[kBins];
  s_hist[threadIdx.x] = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned dmask = (1u << bits) - 1;
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    const int64_t i = item_index(blockIdx.x, warp, lane, it);
    if (i < n) atomicAdd(&s_hist[static_cast<unsigned>(key[i] >> shift) & dmask], 1);
  }
  __syncthreads();
  counts[static_cast<int64_t>(threadIdx.x) * nblocks + blockIdx.x] = s_hist[threadIdx.x];  // digit-major
}

// base[digit * nblocks + block] = first output slot of that CTA's keys with that digit
__global__ void __launch_bounds__(kThreads)
scatter_kernel(const u64* __restrict__ kin, const unsigned* __restrict__ vin, int64_t n, int shift, int bits,
               int nblocks, const int* __restrict__ base, u64* __restrict__ kout, unsigned* __restrict__ vout) {
  __shared__ int s_cnt[kWarps][kBins];  // per-warp digit counts, then first slots
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned dmask = (1u << bits) - 1;
  const unsigned lt = (1u << lane) - 1;
  for (int e = threadIdx.x; e < kWarps * kBins; e += kThreads) (&s_cnt[0][0])[e] = 0;
  __syncthreads();
  u64 k[kItems];
  int rank[kItems];  // among this warp's earlier keys with the same digit
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    const int64_t i = item_index(blockIdx.x, warp, lane, it);
    const bool live = i < n;
    k[it] = live ? kin[i] : 0ull;
    const unsigned d = live ? (static_cast<unsigned>(k[it] >> shift) & dmask) : 0xffffffffu;
    const unsigned same = __match_any_sync(0xffffffffu, d);
    const int leader = __ffs(same) - 1;
    int first = 0;
    if (live && lane == leader) {
      first = s_cnt[warp][d];
      s_cnt[warp][d] = first + __popc(same);
    }
    first = __shfl_sync(0xffffffffu, first, leader);
    rank[it] = first + __popc(same & lt);
    __syncwarp();
  }
  __syncthreads();
  {  // digit = threadIdx.x: warp totals -> first slots (earlier warps of the tile come first)
    const int d = threadIdx.x;
    int run = base[static_cast<int64_t>(d) * nblocks + blockIdx.x];
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const int c = s_cnt[w][d];
      s_cnt[w][d] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    const int64_t i = item_index(blockIdx.x, warp, lane, it);
    if (i < n) {
      const unsigned d = static_cast<unsigned>(k[it] >> shift) & dmask;
      const int dst = s_cnt[warp][d] + rank[it];
      kout[dst] = k[it];
      vout[dst] = vin[i];
    }
  }
}

// ---- one kernel per pass (n < 2^30)
constexpr unsigned kFlagAgg = 1u << 30, kFlagPrefix = 2u << 30, kValueMask = (1u << 30) - 1;
constexpr int kMaxPasses = 8;

// ghist[p * 256 + d] += keys whose digit p is d (zeroed by the caller).
// Shared-memory atomics on a block histogram; a warp whose 32 keys share the
// digit (the usual case for the high digits: segment bits of keys that arrive
// grouped by segment, or constant upper bits) adds once instead of serialising
// 32 ways on one word.
__global__ void __launch_bounds__(kThreads) digit_totals_kernel(const u64* __restrict__ key, int64_t n, int end_bit,
                                                                int passes, unsigned* __restrict__ ghist) {
  __shared__ unsigned s_hist[kMaxPasses * kBins];
  for (int e = threadIdx.x; e < passes * kBins; e += kThreads) s_hist[e] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int64_t b = blockIdx.x * static_cast<int64_t>(kThreads); b < n; b += static_cast<int64_t>(gridDim.x) * kThreads) {
    const int64_t i = b + threadIdx.x;
    const bool live = i < n;  // whole warps per trip: only the last warp of the array is ragged
    const u64 k = live ? low_bits(key[i], end_bit) : 0ull;
    const bool full = __all_sync(0xffffffffu, live);
    for (int p = 0; p < passes; ++p) {
      const unsigned d = static_cast<unsigned>(k >> (8 * p)) & 255u;
      const unsigned d0 = __shfl_sync(0xffffffffu, d, 0);
      if (full && __all_sync(0xffffffffu, d == d0)) {
        if (lane == 0) atomicAdd(&s_hist[p * kBins + d0], 32u);
      } else if (live) {
        atomicAdd(&s_hist[p * kBins + d], 1u);
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < passes * kBins; e += kThreads)
    if (s_hist[e]) atomicAdd(&ghist[e], s_hist[e]);
}

// One pass. ghist: this pass's 256 digit totals; state[tile * 256 + d]: flag |
// count words (zeroed); ticket: this pass's tile counter (zeroed). The tile is
// reordered by digit in shared memory first, so a digit's keys leave as one
// contiguous run (coalesced stores instead of one sector per key).
struct SweepSmem {
  u64 key[kTile];
  unsigned val[kTile];
  int cnt[kWarps][kBins];  // per-warp digit counts, then keys of earlier warps with that digit
  int dstart[kBins];       // first tile-local slot of the digit
  int gofs[kBins];         // global slot = gofs[digit] + tile-local slot
  int scan[32];
  unsigned tile;
};

__global__ void __launch_bounds__(kThreads, 3)
onesweep_kernel(const u64* __restrict__ kin, const unsigned* __restrict__ vin, int64_t n, int shift, int bits,
                const unsigned* __restrict__ ghist, unsigned* state, unsigned* ticket, u64* __restrict__ kout,
                unsigned* __restrict__ vout) {
  extern __shared__ __align__(16) unsigned char sweep_raw[];
  SweepSmem& sm = *reinterpret_cast<SweepSmem*>(sweep_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned dmask = (1u << bits) - 1;
  const unsigned lt = (1u << lane) - 1;
  if (threadIdx.x == 0) sm.tile = atomicAdd(ticket, 1u);
  for (int e = threadIdx.x; e < kWarps * kBins; e += kThreads) (&sm.cnt[0][0])[e] = 0;
  __syncthreads();
  const int64_t tile = sm.tile;
  u64 k[kItems];
  unsigned short rank[kItems];  // among this warp's earlier keys with the same digit (< 512)
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    const int64_t i = item_index(tile, warp, lane, it);
    const bool live = i < n;
    k[it] = live ? kin[i] : 0ull;
    const unsigned d = live ? (static_cast<unsigned>(k[it] >> shift) & dmask) : 0xffffffffu;
    const unsigned same = __match_any_sync(0xffffffffu, d);
    const int leader = __ffs(same) - 1;
    int first = 0;
    if (live && lane == leader) {
      first = sm.cnt[warp][d];
      sm.cnt[warp][d] = first + __popc(same);
    }
    first = __shfl_sync(0xffffffffu, first, leader);
    rank[it] = static_cast<unsigned short>(first + __popc(same & lt));
    __syncwarp();
  }
  __syncthreads();
  {
    const int d = threadIdx.x;
    int total = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const int c = sm.cnt[w][d];
      sm.cnt[w][d] = total;
      total += c;
    }
    volatile unsigned* st = state;
    unsigned before = 0;  // keys of earlier tiles with digit d
    if (tile > 0) {
      st[tile * kBins + d] = kFlagAgg | static_cast<unsigned>(total);
      // look back kLook tiles per trip: the loads are independent, so a walk
      // over many still-running predecessors costs one memory latency per
      // kLook tiles instead of one per tile
      constexpr int kLook = 8;
      bool done = false;
      for (int64_t t = tile - 1; !done; t -= kLook) {
        unsigned v[kLook];
#pragma unroll
        for (int u = 0; u < kLook; ++u) v[u] = t - u >= 0 ? st[(t - u) * kBins + d] : (2u << 30);  // before tile 0: an inclusive prefix of 0
#pragma unroll
        for (int u = 0; u < kLook; ++u) {
          if (!done) {
            unsigned x = v[u];
            while ((x >> 30) == 0) x = st[(t - u) * kBins + d];
            before += x & kValueMask;
            done = (x & kFlagPrefix) != 0;
          }
        }
      }
    }
    st[tile * kBins + d] = kFlagPrefix | (before + static_cast<unsigned>(total));
    int all;
    const int dstart = scan::block_exclusive<int>(total, sm.scan, all);
    __syncthreads();  // sm.scan is reused
    const int smaller = scan::block_exclusive<int>(static_cast<int>(ghist[d]), sm.scan, all);
    sm.dstart[d] = dstart;
    sm.gofs[d] = smaller + static_cast<int>(before) - dstart;
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    const int64_t i = item_index(tile, warp, lane, it);
    if (i < n) {
      const unsigned d = static_cast<unsigned>(k[it] >> shift) & dmask;
      const int slot = sm.dstart[d] + sm.cnt[warp][d] + rank[it];
      sm.key[slot] = k[it];
      sm.val[slot] = vin[i];
    }
  }
  __syncthreads();
  const int64_t left = n - tile * kTile;
  const int live_items = left < kTile ? static_cast<int>(left) : kTile;
#pragma unroll 4
  for (int j = threadIdx.x; j < live_items; j += kThreads) {
    const u64 key = sm.key[j];
    const int dst = sm.gofs[static_cast<unsigned>(key >> shift) & dmask] + j;
    kout[dst] = key;
    vout[dst] = sm.val[j];
  }
}

__global__ void copy_kernel(const u64* __restrict__ kin, const unsigned* __restrict__ vin, int64_t n,
                            u64* __restrict__ kout, unsigned* __restrict__ vout) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    kout[i] = kin[i];
    vout[i] = vin[i];
  }
}

inline int64_t blocks_for(int64_t n) { return (n + kTile - 1) / kTile; }

// bytes of workspace for n pairs: one alternate (key, payload) buffer, the
// (digit, CTA) counts and the scan's block totals
inline size_t workspace_bytes(int64_t n) {
  if (n <= kSmall) return 16;
  const int64_t nb = blocks_for(n), nc = nb * kBins;
  auto up = [](size_t b) { return (b + 255) / 256 * 256; };
  if (n < (1ll << 30))  // tile states of every pass, digit totals, tickets
    return up(n * sizeof(u64)) + up(n * sizeof(unsigned)) +
           up((static_cast<size_t>(kMaxPasses) * nc + kMaxPasses * kBins + kMaxPasses) * sizeof(unsigned));
  return up(n * sizeof(u64)) + up(n * sizeof(unsigned)) + up(nc * sizeof(int)) + up(scan::workspace(nc) * sizeof(int));
}

// (kout, vout) = (kin, vin) stably sorted by the keys' bits [0, end_bit).
// n < 2^31 (positions and slots are ints). `launches` counts the kernels issued.
inline void pairs(const u64* kin, u64* kout, const unsigned* vin, unsigned* vout, int64_t n, int end_bit, void* ws,
                  cudaStream_t stream, int& launches) {
  if (n <= 0) return;
  if (end_bit <= 0) {
    copy_kernel<<<static_cast<unsigned>((n + 255) / 256 > 1184 ? 1184 : (n + 255) / 256), 256, 0, stream>>>(
        kin, vin, n, kout, vout);
    ++launches;
    return;
  }
  if (n <= kSmall) {
    small_kernel<<<1, 1024, 0, stream>>>(kin, vin, static_cast<int>(n), end_bit, kout, vout);
    ++launches;
    return;
  }
  const int64_t nb = blocks_for(n), nc = nb * kBins;
  auto up = [](size_t b) { return (b + 255) / 256 * 256; };
  char* w = static_cast<char*>(ws);
  u64* kalt = reinterpret_cast<u64*>(w);
  w += up(n * sizeof(u64));
  unsigned* valt = reinterpret_cast<unsigned*>(w);
  w += up(n * sizeof(unsigned));
  const int passes = (end_bit + 7) / 8;
  const u64* ksrc = kin;
  const unsigned* vsrc = vin;
  if (n < (1ll << 30)) {
    unsigned* state = reinterpret_cast<unsigned*>(w);          // [passes][nb][256]
    unsigned* ghist = state + static_cast<size_t>(passes) * nc;  // [passes][256]
    unsigned* ticket = ghist + passes * kBins;                  // [passes]
    // per device, so set on every call (a host-side table lookup)
    cudaFuncSetAttribute(onesweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(SweepSmem)));
    cudaMemsetAsync(state, 0, (static_cast<size_t>(passes) * nc + passes * kBins + passes) * sizeof(unsigned), stream);
    const int64_t hb = (n + kThreads * 8 - 1) / (kThreads * 8);
    digit_totals_kernel<<<static_cast<unsigned>(hb > 1184 ? 1184 : hb), kThreads, 0, stream>>>(kin, n, end_bit, passes,
                                                                                              ghist);
    ++launches;
    for (int p = 0; p < passes; ++p) {
      const int shift = 8 * p, bits = end_bit - shift < 8 ? end_bit - shift : 8;
      const bool to_out = ((passes - 1 - p) & 1) == 0;  // the last pass writes (kout, vout)
      u64* kdst = to_out ? kout : kalt;
      unsigned* vdst = to_out ? vout : valt;
      onesweep_kernel<<<static_cast<unsigned>(nb), kThreads, sizeof(SweepSmem), stream>>>(
          ksrc, vsrc, n, shift, bits, ghist + p * kBins, state + static_cast<size_t>(p) * nc, ticket + p, kdst, vdst);
      ++launches;
      ksrc = kdst;
      vsrc = vdst;
    }
    return;
  }
  int* counts = reinterpret_cast<int*>(w);
  w += up(nc * sizeof(int));
  int* scan_ws = reinterpret_cast<int*>(w);
  for (int p = 0; p < passes; ++p) {
    const int shift = 8 * p, bits = end_bit - shift < 8 ? end_bit - shift : 8;
    // the last pass writes (kout, vout): passes - 1 - p even -> out
    const bool to_out = ((passes - 1 - p) & 1) == 0;
    u64* kdst = to_out ? kout : kalt;
    unsigned* vdst = to_out ? vout : valt;
    hist_kernel<<<static_cast<unsigned>(nb), kThreads, 0, stream>>>(ksrc, n, shift, bits, static_cast<int>(nb),
                                                                    counts);
    ++launches;
    scan::exclusive<int>(counts, counts, nc, scan_ws, stream, launches);
    scatter_kernel<<<static_cast<unsigned>(nb), kThreads, 0, stream>>>(ksrc, vsrc, n, shift, bits,
                                                                       static_cast<int>(nb), counts, kdst, vdst);
    ++launches;
    ksrc = kdst;
    vsrc = vdst;
  }
}

}  // namespace sort
}  // namespace liecl_b200
