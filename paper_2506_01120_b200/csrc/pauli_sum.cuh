// Multi-term PauliSum kernels, bit-exact.
//
// A batch holds `nseg` sums as segments of (key, coefficient) arrays, key =
// pauli::pack(x, z) (its numeric order is the reference's (z, x) order,
// PauliStringLess, R:include/liecl/pauli.hpp:41-45). The reference's three
// PauliSum producers on the closure path all end in PauliSum::from_terms
// (R:src/pauli.cpp:78-115): accumulate equal keys in input order into a
// value-initialised slot, drop |c| <= 1e-14 * max |c|, sort. On the device that
// is one "merge": a STABLE segmented sort by key (equal keys keep their input
// order), one thread per run adding the run in order from +0, a per-segment
// max / floor / keep pass and a compaction. The producers:
//   sum_commutator    (R:src/pauli.cpp:179-200): term-pair products, a-major,
//                     commuting pairs skipped, w = a*b, w + w, exact phase;
//   sum_inner_product (:202-220): per basis element, shared keys in sorted
//                     order, acc += conj(v) * h from +0 -- a merge keyed by the
//                     basis index (no drop);
//   linear_combination (R:src/operator.cpp:164-181): base terms times (1, 0),
//                     then every basis element's terms times -beta_l, l
//                     ascending. Elements with beta_l == 0 are skipped: their
//                     products are signed zeros, and a from_terms slot that
//                     starts at +0 can never be changed by adding a zero
//                     (x + -0 = x; +0 + -0 = +0), nor can a zero move the max.
// Every arithmetic step uses the explicitly rounded intrinsics of pauli.cuh
// (no FMA contraction), so coefficients are the reference's bits. The drop
// test uses CUDA hypot for std::abs (glibc cabs); both are faithful, so they
// could only disagree for a coefficient within an ulp of 1e-14 * max.
#pragma once

#include "common.cuh"
#include "pauli.cuh"

namespace liecl_b200 {
namespace psum {

using pauli::C2;
using pauli::cadd;
using pauli::cmul;
constexpr double kDropTolerance = 1e-14;  // R:include/liecl/pauli.hpp:73

// ---- string keys -------------------------------------------------------------
// Every kernel below is a template over the key type K:
//  * narrow (1..31 qubits): unsigned long long x | z << 32, whose numeric
//    order is the reference's (z, x) order (PauliStringLess);
//  * wide (32..64 qubits): WKey {x, z}, ordered by (z, x).
// Both reserve all ones as the marker of a commuting product (sorts last) and
// of a free hash slot; no string of <= 63 qubits reaches it. Index keys (basis
// element l, the beta merges) live in the same arrays (kfrom_index / kindex).
struct __align__(16) WKey {
  unsigned long long x, z;
};

__host__ __device__ __forceinline__ uint64_t kx(unsigned long long k) { return k & 0xffffffffull; }
__host__ __device__ __forceinline__ uint64_t kz(unsigned long long k) { return k >> 32; }
__host__ __device__ __forceinline__ uint64_t kx(const WKey& k) { return k.x; }
__host__ __device__ __forceinline__ uint64_t kz(const WKey& k) { return k.z; }
__host__ __device__ __forceinline__ bool keq(unsigned long long a, unsigned long long b) { return a == b; }
__host__ __device__ __forceinline__ bool keq(const WKey& a, const WKey& b) { return a.x == b.x && a.z == b.z; }
__host__ __device__ __forceinline__ bool kless(unsigned long long a, unsigned long long b) { return a < b; }
__host__ __device__ __forceinline__ bool kless(const WKey& a, const WKey& b) {
  return a.z < b.z || (a.z == b.z && a.x < b.x);
}
__host__ __device__ __forceinline__ unsigned long long kxor(unsigned long long a, unsigned long long b) { return a ^ b; }
__host__ __device__ __forceinline__ WKey kxor(const WKey& a, const WKey& b) { return {a.x ^ b.x, a.z ^ b.z}; }
__host__ __device__ __forceinline__ bool kmarked(unsigned long long k) { return k == ~0ull; }
__host__ __device__ __forceinline__ bool kmarked(const WKey& k) { return (k.x & k.z) == ~0ull; }
__host__ __device__ __forceinline__ int64_t kindex(unsigned long long k) { return static_cast<int64_t>(k); }
__host__ __device__ __forceinline__ int64_t kindex(const WKey& k) { return static_cast<int64_t>(k.x); }
__device__ __forceinline__ uint64_t khash(unsigned long long k) { return pauli::mix(k); }
__device__ __forceinline__ uint64_t khash(const WKey& k) { return pauli::mix2(k.x, k.z); }
__device__ __forceinline__ unsigned long long kcas(unsigned long long* p, unsigned long long cmp,
                                                   unsigned long long v) {
  return atomicCAS(p, cmp, v);
}
__device__ __forceinline__ WKey kcas(WKey* p, WKey cmp, WKey v) {
  const unsigned __int128 c = (static_cast<unsigned __int128>(cmp.z) << 64) | cmp.x;
  const unsigned __int128 w = (static_cast<unsigned __int128>(v.z) << 64) | v.x;
  const unsigned __int128 r = atomicCAS(reinterpret_cast<unsigned __int128*>(p), c, w);
  return {static_cast<unsigned long long>(r), static_cast<unsigned long long>(r >> 64)};
}
template <class K> __host__ __device__ __forceinline__ K kpack(uint64_t x, uint64_t z);
template <> __host__ __device__ __forceinline__ unsigned long long kpack<unsigned long long>(uint64_t x, uint64_t z) {
  return static_cast<unsigned long long>(x) | (static_cast<unsigned long long>(z) << 32);
}
template <> __host__ __device__ __forceinline__ WKey kpack<WKey>(uint64_t x, uint64_t z) { return {x, z}; }
template <class K> __host__ __device__ __forceinline__ K kmarker() { return kpack<K>(~0ull, ~0ull) ; }
template <> __host__ __device__ __forceinline__ unsigned long long kmarker<unsigned long long>() { return ~0ull; }
template <class K> __host__ __device__ __forceinline__ K kfrom_index(int64_t l);
template <> __host__ __device__ __forceinline__ unsigned long long kfrom_index<unsigned long long>(int64_t l) {
  return static_cast<unsigned long long>(l);
}
template <> __host__ __device__ __forceinline__ WKey kfrom_index<WKey>(int64_t l) {
  return {static_cast<unsigned long long>(l), 0ull};
}

// Bracket products of cursor pairs [g0, g0 + cnt): one block per pair,
// product q = ia * |b| + ib at off[p] + q (a = basis[l], b = basis[m]).
template <class K>
__global__ void products_kernel(int64_t g0, int cnt, const int* __restrict__ off, const int64_t* __restrict__ boff,
                                const K* __restrict__ bkey, const C2* __restrict__ bval, K* __restrict__ out_key,
                                C2* __restrict__ out_val, int* __restrict__ marker_flag) {
  const int p = blockIdx.x;
  if (p >= cnt) return;
  int64_t l, m;
  pair_from_index(g0 + p, l, m);
  const int64_t a0 = boff[l], na = boff[l + 1] - a0;
  const int64_t b0 = boff[m], nb = boff[m + 1] - b0;
  const int base = off[p];
  for (int64_t q = threadIdx.x; q < na * nb; q += blockDim.x) {
    const int64_t ia = q / nb, ib = q - ia * nb;
    const K ka = bkey[a0 + ia], kb = bkey[b0 + ib];
    const uint64_t xa = kx(ka), za = kz(ka), xb = kx(kb), zb = kz(kb);
    K key = kmarker<K>();
    C2 w{0.0, 0.0};
    if (!pauli::commute(xa, za, xb, zb)) {
      w = cmul(bval[a0 + ia], bval[b0 + ib]);
      w = pauli::apply_phase(cadd(w, w), pauli::phase_exponent(xa, za, xb, zb));
      key = kxor(ka, kb);
      if (marker_flag && kmarked(key)) *marker_flag = 1;  // 64 qubits: the product is Y^64 (sum_engine.cuh)
    }
    out_key[base + q] = key;
    out_val[base + q] = w;
  }
}

__global__ void iota_kernel(unsigned* __restrict__ idx, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) idx[i] = i;
}

// seg[i] = the segment holding position i (largest p with off[p] <= i)
__global__ void seg_of_kernel(const int* __restrict__ off, int nseg, int n, int* __restrict__ seg) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int lo = 0, hi = nseg - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (off[mid] <= i) lo = mid;
      else hi = mid - 1;
    }
    seg[i] = lo;
  }
}

// Combined sort key (segment | invalid | key) for one stable LSD radix sort of
// the whole batch over only its live bits: Pauli keys compact to 2q bits
// x | z << q (the (z, x) order is kept), index keys (basis l) use kbits bits.
template <class K>
__global__ void combine_kernel(const int* __restrict__ off, int nseg, int n, const K* __restrict__ key, int pauli_q,
                               int kbits, unsigned long long* __restrict__ ck) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int lo = 0, hi = nseg - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (off[mid] <= i) lo = mid;
      else hi = mid - 1;
    }
    const K k = key[i];
    unsigned long long c;
    if (pauli_q > 0) {
      c = kmarked(k) ? (1ull << kbits) : (kx(k) | (kz(k) << pauli_q));
    } else {
      c = static_cast<unsigned long long>(kindex(k));
    }
    ck[i] = (static_cast<unsigned long long>(lo) << (kbits + 1)) | c;
  }
}
template <class K>
__global__ void split_kernel(const unsigned long long* __restrict__ ck, int n, int pauli_q, int kbits,
                             K* __restrict__ ks, int* __restrict__ seg) {
  const unsigned long long kmask = (1ull << kbits) - 1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned long long c = ck[i];
    seg[i] = static_cast<int>(c >> (kbits + 1));
    if ((c >> kbits) & 1ull) {
      ks[i] = kmarker<K>();
    } else if (pauli_q > 0) {
      const unsigned long long k = c & kmask, qm = (1ull << pauli_q) - 1;
      ks[i] = kpack<K>(k & qm, k >> pauli_q);
    } else {
      ks[i] = kfrom_index<K>(static_cast<int64_t>(c & kmask));
    }
  }
}

// first element of each (segment, key) run of the sorted keys
template <class K>
__global__ void heads_kernel(const K* __restrict__ ks, const int* __restrict__ seg, int n, int* __restrict__ flag) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    flag[i] = !kmarked(ks[i]) && (i == 0 || seg[i] != seg[i - 1] || !keq(ks[i], ks[i - 1]));
}

// from_terms accumulation: each run summed in input order from +0
template <class K>
__global__ void run_sum_kernel(const K* __restrict__ ks, const unsigned* __restrict__ is, const C2* __restrict__ val,
                               const int* __restrict__ seg, const int* __restrict__ flag, const int* __restrict__ pos,
                               int n, K* __restrict__ rkey, C2* __restrict__ rval, double* __restrict__ rmag,
                               int* __restrict__ rseg) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (!flag[i]) continue;
    const K k = ks[i];
    const int sgi = seg[i];
    C2 acc = pauli::slot(val[is[i]]);
    // the run's terms are added in input order (from_terms' order); the loads
    // of the next kAhead entries are issued together so a long run costs one
    // memory latency per kAhead terms, not two per term (entries past the
    // run's end are loaded and dropped: they are inside the arrays)
    constexpr int kAhead = 8;
    int j = i + 1;
    // most runs are one term long: look at the next entry alone first
    if (j < n && keq(ks[j], k) && seg[j] == sgi) acc = cadd(acc, val[is[j]]), ++j;
    else j = n;
    for (; j < n;) {
      const int m = n - j < kAhead ? n - j : kAhead;
      K kk[kAhead];
      int sg[kAhead];
      C2 vv[kAhead];
#pragma unroll
      for (int u = 0; u < kAhead; ++u)
        if (u < m) {
          kk[u] = ks[j + u];
          sg[u] = seg[j + u];
          vv[u] = val[is[j + u]];
        }
      int u = 0;
#pragma unroll
      for (int q = 0; q < kAhead; ++q)
        if (u == q && q < m && keq(kk[q], k) && sg[q] == sgi) {
          acc = cadd(acc, vv[q]);
          ++u;
        }
      if (u < m) break;
      j += m;
    }
    const int r = pos[i];
    rkey[r] = k;
    rval[r] = acc;
    rmag[r] = hypot(acc.re, acc.im);
    rseg[r] = sgi;
  }
}

// out[p] = pos[off[p]] (positions before segment p), total past the end
__global__ void seg_positions_kernel(const int* __restrict__ off, int nseg, int n, const int* __restrict__ pos,
                                     int total, int* __restrict__ out) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p <= nseg; p += gridDim.x * blockDim.x)
    out[p] = (p < nseg && off[p] < n) ? pos[off[p]] : total;
}

// drop rule per segment: keep |c| > 1e-14 * max |c| (one warp per segment)
__global__ void floor_keep_kernel(const int* __restrict__ roff, int nseg, const double* __restrict__ rmag,
                                  int* __restrict__ keep) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= nseg) return;
  const int b = roff[warp], e = roff[warp + 1];
  double mx = 0.0;
  for (int r = b + lane; r < e; r += 32) mx = fmax(mx, rmag[r]);
  for (int s = 16; s > 0; s >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, s));
  const double floor = __dmul_rn(kDropTolerance, mx);
  for (int r = b + lane; r < e; r += 32) keep[r] = rmag[r] > floor;
}

template <class K>
__global__ void compact_kernel(const int* __restrict__ keep, const int* __restrict__ kpos, int n,
                               const K* __restrict__ rkey, const C2* __restrict__ rval, K* __restrict__ okey,
                               C2* __restrict__ oval) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    if (keep[r]) {
      okey[kpos[r]] = rkey[r];
      oval[kpos[r]] = rval[r];
    }
}

// sqrt(sum_t std::norm(c_t)) in term order (sum_norm, R:src/pauli.cpp:222-228)
__global__ void seg_norm_kernel(const int* __restrict__ off, int nseg, const C2* __restrict__ val,
                                double* __restrict__ out) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < nseg; p += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int t = off[p]; t < off[p + 1]; ++t)
      acc = __dadd_rn(acc, __dadd_rn(__dmul_rn(val[t].re, val[t].re), __dmul_rn(val[t].im, val[t].im)));
    out[p] = __dsqrt_rn(acc);
  }
}

// Complex{1/norm, 0} * sum for segments with norm > tol (R:src/closure.cpp:419-423)
__global__ void seg_scale_kernel(const int* __restrict__ off, int nseg, const double* __restrict__ nrm, double tol,
                                 C2* __restrict__ val) {
  for (int p = blockIdx.x; p < nseg; p += gridDim.x) {
    if (!(nrm[p] > tol)) continue;
    const C2 s{__ddiv_rn(1.0, nrm[p]), 0.0};
    for (int t = off[p] + threadIdx.x; t < off[p + 1]; t += blockDim.x) val[t] = cmul(val[t], s);
  }
}

// ---- key -> (basis index, coefficient) lists, ascending basis index -------

template <class K> struct Index {
  K* key;  // open-addressed slots (kmarker = free)
  int* head;
  int* tail;
  int* count;
  uint64_t mask;
  int* e_l;  // entries, appended in accept order (so every list is ascending in l)
  C2* e_v;
  int* e_next;
};

template <class K> __device__ __forceinline__ int index_find(const Index<K>& ix, const K& key) {
  for (uint64_t p = khash(key) & ix.mask;; p = (p + 1) & ix.mask) {
    const K k = ix.key[p];
    if (keq(k, key)) return static_cast<int>(p);
    if (kmarked(k)) return -1;
  }
}

// Append the n terms (distinct keys) of accepted element l as entries e0...
template <class K>
__global__ void index_insert_kernel(Index<K> ix, const K* __restrict__ key, const C2* __restrict__ val, int n, int l,
                                    int e0) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int e = e0 + t;
    ix.e_l[e] = l;
    ix.e_v[e] = val[t];
    ix.e_next[e] = -1;
    const K k = key[t];
    for (uint64_t p = khash(k) & ix.mask;; p = (p + 1) & ix.mask) {
      const K prev = kcas(&ix.key[p], kmarker<K>(), k);
      if (kmarked(prev)) {
        ix.head[p] = e;
        ix.tail[p] = e;
        ix.count[p] = 1;
        break;
      }
      if (keq(prev, k)) {  // one thread per key in this launch
        ix.e_next[ix.tail[p]] = e;
        ix.tail[p] = e;
        ix.count[p] += 1;
        break;
      }
    }
  }
}

// move every occupied slot of `from` into `to` (lists unchanged)
template <class K> __global__ void index_rehash_kernel(Index<K> from, uint64_t from_slots, Index<K> to) {
  for (uint64_t s = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; s < from_slots;
       s += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const K k = from.key[s];
    if (kmarked(k)) continue;
    for (uint64_t p = khash(k) & to.mask;; p = (p + 1) & to.mask) {
      if (kmarked(kcas(&to.key[p], kmarker<K>(), k))) {
        to.head[p] = from.head[s];
        to.tail[p] = from.tail[s];
        to.count[p] = from.count[s];
        break;
      }
    }
  }
}

template <class K> __global__ void index_reset_kernel(Index<K> ix, uint64_t slots) {
  for (uint64_t s = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; s < slots;
       s += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    ix.key[s] = kmarker<K>();
}

// overlap contributions of each term: one per basis element l < n_limit that
// holds the term's string
template <class K>
__global__ void beta_count_kernel(Index<K> ix, const K* __restrict__ key, int n, int n_limit,
                                  long long* __restrict__ cnt) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int s = index_find(ix, key[t]);
    long long c = 0;
    if (s >= 0)
      for (int e = ix.head[s]; e >= 0 && ix.e_l[e] < n_limit; e = ix.e_next[e]) ++c;
    cnt[t] = c;
  }
}
// (l, conj(v_l) * h_t) at pos[t].. in ascending l; the segment's terms are in
// sorted key order, so a stable sort by l leaves each l's contributions in
// the order sum_inner_product adds them
template <class K>
__global__ void beta_fill_kernel(Index<K> ix, const K* __restrict__ key, const C2* __restrict__ val, int n,
                                 int n_limit, const long long* __restrict__ pos, K* __restrict__ out_l,
                                 C2* __restrict__ out_v) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int s = index_find(ix, key[t]);
    if (s < 0) continue;
    long long w = pos[t];
    for (int e = ix.head[s]; e >= 0 && ix.e_l[e] < n_limit; e = ix.e_next[e], ++w) {
      const C2 v = ix.e_v[e];
      out_l[w] = kfrom_index<K>(ix.e_l[e]);
      out_v[w] = cmul({v.re, -v.im}, val[t]);
    }
  }
}

// linear_combination chunks: segment p's base chunk sits at p + broff[p], its
// beta runs r (segment p) at r + p + 1
struct Chunk {
  int len;
  int kind;  // 0: base (segment terms), 1: basis element
  int64_t src;
  C2 mult;
};
__global__ void chunk_base_kernel(const int* __restrict__ hoff, const int* __restrict__ broff, int nseg, C2 base,
                                  Chunk* __restrict__ ch, long long* __restrict__ clen) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < nseg; p += gridDim.x * blockDim.x) {
    const int k = p + broff[p];
    ch[k] = {hoff[p + 1] - hoff[p], 0, hoff[p], base};
    clen[k] = ch[k].len;
  }
}
template <class K>
__global__ void chunk_basis_kernel(const K* __restrict__ bl, const C2* __restrict__ beta,
                                   const int* __restrict__ rseg, int nruns, const int64_t* __restrict__ voff,
                                   bool negate, Chunk* __restrict__ ch, long long* __restrict__ clen) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nruns; r += gridDim.x * blockDim.x) {
    const int k = r + rseg[r] + 1;
    const int64_t l = kindex(bl[r]);
    const C2 b = beta[r];
    const bool zero = b.re == 0.0 && b.im == 0.0;
    ch[k] = {zero ? 0 : static_cast<int>(voff[l + 1] - voff[l]), 1, voff[l],
             negate ? C2{-b.re, -b.im} : b};
    clen[k] = ch[k].len;
  }
}
// one block per chunk: coefficient = mult * term (base_coeff * t, coeffs[l] * t)
template <class K>
__global__ void chunk_fill_kernel(const Chunk* __restrict__ ch, const long long* __restrict__ cpos, int nchunks,
                                  const K* __restrict__ hkey, const C2* __restrict__ hval, const K* __restrict__ vkey,
                                  const C2* __restrict__ vval, K* __restrict__ out_key, C2* __restrict__ out_val) {
  for (int k = blockIdx.x; k < nchunks; k += gridDim.x) {
    const Chunk c = ch[k];
    const K* sk = (c.kind == 0 ? hkey : vkey) + c.src;
    const C2* sv = (c.kind == 0 ? hval : vval) + c.src;
    for (int t = threadIdx.x; t < c.len; t += blockDim.x) {
      out_key[cpos[k] + t] = sk[t];
      out_val[cpos[k] + t] = cmul(c.mult, sv[t]);
    }
  }
}

// int segment offsets from 64-bit exclusive-scan positions:
// out[p] = pos[first item of segment p] (items = the segment's first chunk
// when `chunked`, else its first term), total past the end
__global__ void seg_offsets64_kernel(const int* __restrict__ off, const int* __restrict__ broff, int nseg, int n,
                                     const long long* __restrict__ pos, long long total, int* __restrict__ out) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p <= nseg; p += gridDim.x * blockDim.x) {
    if (p == nseg) {
      out[p] = static_cast<int>(total);
      continue;
    }
    const int item = broff ? p + broff[p] : off[p];
    out[p] = item < n ? static_cast<int>(pos[item]) : static_cast<int>(total);
  }
}

__global__ void rebase_kernel(const int* __restrict__ off, int a, int nseg, int* __restrict__ out) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p <= nseg; p += gridDim.x * blockDim.x) out[p] = off[a + p] - off[a];
}

// accept: Complex{1/rn, 0} * residual -> pool (R:src/closure.cpp:287-290)
template <class K>
__global__ void append_scaled_kernel(const K* __restrict__ key, const C2* __restrict__ val, int n, double rn,
                                     K* __restrict__ okey, C2* __restrict__ oval) {
  const C2 s{__ddiv_rn(1.0, rn), 0.0};
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    okey[t] = key[t];
    oval[t] = cmul(val[t], s);
  }
}

// PauliSum::operator*(Complex) (R:src/pauli.cpp:166-177): t.coefficient * scalar
__global__ void scale_terms_kernel(C2* __restrict__ v, int64_t n, C2 s) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x)
    v[t] = cmul(v[t], s);
}

// Alg. 2 on sums: per-segment overlap runs (l, beta) -> dense column-major
// n x nseg (zeroed first), and a dense n x nseg coefficient block -> runs
// (every l of every segment; chunk_basis_kernel skips exact zeros)
template <class K>
__global__ void scatter_runs_kernel(const K* __restrict__ key, const C2* __restrict__ val, const int* __restrict__ rseg,
                                    int nruns, int64_t ld, C2* __restrict__ out) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nruns; r += gridDim.x * blockDim.x)
    out[static_cast<int64_t>(rseg[r]) * ld + kindex(key[r])] = val[r];
}
template <class K>
__global__ void dense_runs_kernel(const C2* __restrict__ X, int n, int nseg, K* __restrict__ key, C2* __restrict__ val,
                                  int* __restrict__ rseg, int* __restrict__ off) {
  const int64_t total = static_cast<int64_t>(n) * nseg;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    key[e] = kfrom_index<K>(e % n);
    val[e] = X[e];
    rseg[e] = static_cast<int>(e / n);
  }
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p <= nseg;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x)
    off[p] = static_cast<int>(p * n);
}

} // namespace psum
} // namespace liecl_b200

namespace liecl_b200 {
namespace psum {

// ---- fused single-candidate check (small sums) ------------------------------
// One CTA runs OrthonormStrategy::check for one candidate entirely in shared
// memory: two linear_combination passes (R:src/closure.cpp:142-162) and the
// residual norm. Same arithmetic, same order as the multi-kernel merges:
//  - beta_l: every term's (l, conj(v) h_t) contributions are listed in term
//    order (sorted keys), then one thread adds them from +0 per l in list
//    order -- sum_inner_product's order;
//  - the residual: sources merged one after another (the base terms, then
//    V_l * -beta_l for l ascending); keys are distinct inside a source, so a
//    source is merged in parallel (one thread per key owns its slot) and a
//    barrier separates sources: every slot adds in the reference's order from
//    +0 (PauliSum::from_terms);
//  - drop |c| <= 1e-14 max |c|, bitonic sort of the survivors by key, norm
//    summed in sorted order.
// A candidate whose sums outgrow the shared buffers reports status 1 and the
// engine re-runs the batch through the general merges.
constexpr int kFusedThreads = 256;

template <class K> struct FusedSmem {
  K* hkey;  // open-addressed accumulation slots [hc]
  C2* hval;
  K* skey;  // sorted pass input / output [hc]
  C2* sval;
  K* ckey;  // beta contributions: basis index [hc]
  C2* cval;
  C2* beta;                  // [nb]
  unsigned* touched;         // [nb / 32 + 1]
};

template <class K> __device__ __forceinline__ void fused_bitonic(K* key, C2* val, int count, int npow2) {
  for (int i = count + threadIdx.x; i < npow2; i += blockDim.x) key[i] = kmarker<K>();
  __syncthreads();
  for (int k = 2; k <= npow2; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < npow2; i += blockDim.x) {
        const int p = i ^ j;
        if (p > i) {
          const bool up = (i & k) == 0;
          if (kless(key[p], key[i]) == up) {
            const K tk = key[i];
            key[i] = key[p];
            key[p] = tk;
            const C2 tv = val[i];
            val[i] = val[p];
            val[p] = tv;
          }
        }
      }
      __syncthreads();
    }
}

// one pass: input = (s.skey, s.sval, n_in) sorted; output replaces it; returns
// the output count or -1 on overflow
template <class K>
__device__ int fused_pass(const FusedSmem<K>& s, int hc, int n_in, const Index<K>& ix, int n_limit,
                          const int64_t* __restrict__ voff, const K* __restrict__ vkey, const C2* __restrict__ vval,
                          int* s_scratch) {
  int* s_count = s_scratch;      // [0] contributions, [1] distinct keys, [2] kept, [3] overflow
  int* s_pos = s_scratch + 4;    // per-term contribution offsets [kFusedThreads + 1] chunk scan
  for (int l = threadIdx.x; l < n_limit; l += blockDim.x) s.beta[l] = {0.0, 0.0};
  for (int w = threadIdx.x; w < n_limit / 32 + 1; w += blockDim.x) s.touched[w] = 0u;
  for (int i = threadIdx.x; i < hc; i += blockDim.x) s.hkey[i] = kmarker<K>();
  if (threadIdx.x < 4) s_count[threadIdx.x] = 0;
  __syncthreads();
  // (a) contributions, term-major: chunks of blockDim terms, each chunk
  // scanned so the list keeps term order
  for (int t0 = 0; t0 < n_in; t0 += blockDim.x) {
    const int t = t0 + threadIdx.x;
    int sl = -1, c = 0;
    if (t < n_in) {
      sl = index_find(ix, s.skey[t]);
      if (sl >= 0)
        for (int e = ix.head[sl]; e >= 0 && ix.e_l[e] < n_limit; e = ix.e_next[e]) ++c;
    }
    s_pos[threadIdx.x] = c;
    __syncthreads();
    if (threadIdx.x == 0) {  // exclusive scan of the chunk's counts
      int acc = s_count[0];
      for (int i = 0; i < blockDim.x; ++i) {
        const int v = s_pos[i];
        s_pos[i] = acc;
        acc += v;
      }
      s_count[0] = acc;
      if (acc > hc) s_count[3] = 1;
    }
    __syncthreads();
    if (s_count[3]) return -1;
    if (sl >= 0) {
      int w = s_pos[threadIdx.x];
      const C2 h = s.sval[t];
      for (int e = ix.head[sl]; e >= 0 && ix.e_l[e] < n_limit; e = ix.e_next[e], ++w) {
        const C2 v = ix.e_v[e];
        s.ckey[w] = kfrom_index<K>(ix.e_l[e]);
        s.cval[w] = cmul({v.re, -v.im}, h);
      }
    }
    __syncthreads();
  }
  // (b) beta_l += contributions in list order, from +0
  if (threadIdx.x == 0) {
    for (int i = 0; i < s_count[0]; ++i) {
      const int l = static_cast<int>(kindex(s.ckey[i]));
      s.beta[l] = cadd(s.beta[l], s.cval[i]);
      s.touched[l >> 5] |= 1u << (l & 31);
    }
  }
  __syncthreads();
  // (c) residual slots: the base terms (x (1, 0)), then V_l * -beta_l
  // keys are distinct inside a source, so each key's slot has one writer per
  // source; a new key first reserves capacity (<= 3/4 of the table, the
  // spare quarter >= one CTA of in-flight claims), so probing always ends
  const int limit = (hc * 3) / 4;
  auto merge_source = [&](const K* key, const C2* val, int n, C2 mult) {
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
      const K k = key[t];
      const C2 v = cmul(mult, val[t]);
      for (uint64_t p = khash(k) & static_cast<uint64_t>(hc - 1);; p = (p + 1) & static_cast<uint64_t>(hc - 1)) {
        const K cur = s.hkey[p];
        if (keq(cur, k)) {
          s.hval[p] = cadd(s.hval[p], v);
          break;
        }
        if (!kmarked(cur)) continue;
        const K prev = kcas(&s.hkey[p], kmarker<K>(), k);
        if (kmarked(prev)) {
          if (atomicAdd(&s_count[1], 1) >= limit) s_count[3] = 1;
          s.hval[p] = pauli::slot(v);
          break;
        }
        if (keq(prev, k)) {  // cannot happen within one source; kept for safety
          s.hval[p] = cadd(s.hval[p], v);
          break;
        }
      }
    }
    __syncthreads();
  };
  merge_source(s.skey, s.sval, n_in, {1.0, 0.0});
  for (int w = 0; w < n_limit / 32 + 1 && !s_count[3]; ++w) {
    unsigned bits = s.touched[w];
    while (bits) {
      const int l = w * 32 + __ffs(bits) - 1;
      bits &= bits - 1;
      const C2 b = s.beta[l];
      if (b.re == 0.0 && b.im == 0.0) continue;  // zero products change no slot
      merge_source(vkey + voff[l], vval + voff[l], static_cast<int>(voff[l + 1] - voff[l]), {-b.re, -b.im});
      if (s_count[3]) break;
    }
  }
  if (s_count[3]) return -1;
  // (d) drop rule, compaction, sort
  __shared__ double s_max[kFusedThreads / 32];
  double mx = 0.0;
  for (int i = threadIdx.x; i < hc; i += blockDim.x)
    if (!kmarked(s.hkey[i])) mx = fmax(mx, hypot(s.hval[i].re, s.hval[i].im));
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int i = 0; i < kFusedThreads / 32; ++i) m = fmax(m, s_max[i]);
    s_max[0] = m;
  }
  __syncthreads();
  const double floor = __dmul_rn(kDropTolerance, s_max[0]);
  for (int i = threadIdx.x; i < hc; i += blockDim.x)
    if (!kmarked(s.hkey[i]) && hypot(s.hval[i].re, s.hval[i].im) > floor) {
      const int w = atomicAdd(&s_count[2], 1);
      s.skey[w] = s.hkey[i];
      s.sval[w] = s.hval[i];
    }
  __syncthreads();
  const int nk = s_count[2];
  int np2 = 1;
  while (np2 < nk) np2 <<= 1;
  fused_bitonic(s.skey, s.sval, nk, np2);
  return nk;
}

// OrthonormStrategy::check of segment p of h against basis elements l < n_limit
template <class K>
__global__ void __launch_bounds__(kFusedThreads)
fused_check_kernel(const int* __restrict__ off, int nseg, const K* __restrict__ hkey, const C2* __restrict__ hval,
                   Index<K> ix, int n_limit, const int64_t* __restrict__ voff, const K* __restrict__ vkey,
                   const C2* __restrict__ vval, int hc, K* __restrict__ okey, C2* __restrict__ oval,
                   int* __restrict__ olen, double* __restrict__ rn, int* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char s_raw[];
  __shared__ int s_scratch[4 + kFusedThreads];
  FusedSmem<K> s;
  s.hkey = reinterpret_cast<K*>(s_raw);
  s.skey = s.hkey + hc;
  s.ckey = s.skey + hc;
  s.hval = reinterpret_cast<C2*>(s.ckey + hc);
  s.sval = s.hval + hc;
  s.cval = s.sval + hc;
  s.beta = s.cval + hc;
  s.touched = reinterpret_cast<unsigned*>(s.beta + n_limit);
  for (int p = blockIdx.x; p < nseg; p += gridDim.x) {
    const int b0 = off[p], n_in = off[p + 1] - b0;
    if (n_in > hc) {  // the input alone does not fit
      if (threadIdx.x == 0) status[p] = 1;
      continue;
    }
    for (int t = threadIdx.x; t < n_in; t += blockDim.x) {
      s.skey[t] = hkey[b0 + t];
      s.sval[t] = hval[b0 + t];
    }
    __syncthreads();
    int n = n_in;
    if (n_limit > 0) {  // project_residual of an empty tuple returns h itself
      n = fused_pass(s, hc, n, ix, n_limit, voff, vkey, vval, s_scratch);
      if (n > 0) n = fused_pass(s, hc, n, ix, n_limit, voff, vkey, vval, s_scratch);
    }
    if (n < 0) {
      if (threadIdx.x == 0) status[p] = 1;
      __syncthreads();
      continue;
    }
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
      okey[static_cast<int64_t>(p) * hc + t] = s.skey[t];
      oval[static_cast<int64_t>(p) * hc + t] = s.sval[t];
    }
    if (threadIdx.x == 0) {
      double acc = 0.0;  // sum_norm in term order
      for (int t = 0; t < n; ++t)
        acc = __dadd_rn(acc, __dadd_rn(__dmul_rn(s.sval[t].re, s.sval[t].re), __dmul_rn(s.sval[t].im, s.sval[t].im)));
      rn[p] = __dsqrt_rn(acc);
      olen[p] = n;
      status[p] = 0;
    }
    __syncthreads();
  }
}

// segments starting at src[q] (lengths from off) -> contiguous batch
template <class K>
__global__ void gather_segs_kernel(const K* __restrict__ key, const C2* __restrict__ val, const int* __restrict__ src,
                                   const int* __restrict__ off, int nseg, K* __restrict__ okey, C2* __restrict__ oval) {
  for (int q = blockIdx.x; q < nseg; q += gridDim.x)
    for (int t = threadIdx.x; t < off[q + 1] - off[q]; t += blockDim.x) {
      okey[off[q] + t] = key[src[q] + t];
      oval[off[q] + t] = val[src[q] + t];
    }
}

// strided fused outputs (row p at p * hc) -> contiguous segments
template <class K>
__global__ void strided_to_segs_kernel(const K* __restrict__ sk, const C2* __restrict__ sv, int hc,
                                       const int* __restrict__ off, int nseg, K* __restrict__ ok, C2* __restrict__ ov) {
  for (int p = blockIdx.x; p < nseg; p += gridDim.x)
    for (int t = threadIdx.x; t < off[p + 1] - off[p]; t += blockDim.x) {
      ok[off[p] + t] = sk[static_cast<int64_t>(p) * hc + t];
      ov[off[p] + t] = sv[static_cast<int64_t>(p) * hc + t];
    }
}

template <class K> inline size_t fused_smem_bytes(int hc, int n_limit) {
  return static_cast<size_t>(hc) * 3 * (sizeof(K) + sizeof(C2)) +
         static_cast<size_t>(n_limit) * sizeof(C2) + (static_cast<size_t>(n_limit) / 32 + 1) * sizeof(unsigned);
}

} // namespace psum
} // namespace liecl_b200

namespace liecl_b200 {
namespace psum {

// sort words of the merge's multi-pass path (sum_engine.cuh merge): word w of
// the key at input position perm[i] (wide keys: 0 = x, 1 = z; narrow keys:
// the packed key itself)
template <class K>
__global__ void key_words_kernel(const K* __restrict__ key, const unsigned* __restrict__ perm, int n, int word,
                                 unsigned long long* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const K k = key[perm ? perm[i] : i];
    if constexpr (std::is_same_v<K, WKey>) out[i] = word ? k.z : k.x;
    else out[i] = static_cast<unsigned long long>(k);
  }
}
// the segment holding input position perm[i]
__global__ void seg_words_kernel(const int* __restrict__ off, int nseg, const unsigned* __restrict__ perm, int n,
                                 unsigned long long* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int p = static_cast<int>(perm[i]);
    int lo = 0, hi = nseg - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (off[mid] <= p) lo = mid;
      else hi = mid - 1;
    }
    out[i] = static_cast<unsigned long long>(lo);
  }
}
template <class K>
__global__ void gather_keys_kernel(const K* __restrict__ key, const unsigned* __restrict__ perm, int n,
                                   K* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = key[perm[i]];
}

} // namespace psum
} // namespace liecl_b200
