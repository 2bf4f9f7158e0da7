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
constexpr unsigned long long kInvalid = ~0ull;  // commuting product (sorts last)
constexpr double kDropTolerance = 1e-14;       // R:include/liecl/pauli.hpp:73

__device__ __forceinline__ uint64_t key_x(unsigned long long k) { return k & 0xffffffffull; }
__device__ __forceinline__ uint64_t key_z(unsigned long long k) { return k >> 32; }

// Bracket products of cursor pairs [g0, g0 + cnt): one block per pair,
// product q = ia * |b| + ib at off[p] + q (a = basis[l], b = basis[m]).
__global__ void products_kernel(int64_t g0, int cnt, const int* __restrict__ off, const int64_t* __restrict__ boff,
                                const unsigned long long* __restrict__ bkey, const C2* __restrict__ bval,
                                unsigned long long* __restrict__ out_key, C2* __restrict__ out_val) {
  const int p = blockIdx.x;
  if (p >= cnt) return;
  int64_t l, m;
  pair_from_index(g0 + p, l, m);
  const int64_t a0 = boff[l], na = boff[l + 1] - a0;
  const int64_t b0 = boff[m], nb = boff[m + 1] - b0;
  const int base = off[p];
  for (int64_t q = threadIdx.x; q < na * nb; q += blockDim.x) {
    const int64_t ia = q / nb, ib = q - ia * nb;
    const unsigned long long ka = bkey[a0 + ia], kb = bkey[b0 + ib];
    const uint64_t xa = key_x(ka), za = key_z(ka), xb = key_x(kb), zb = key_z(kb);
    unsigned long long key = kInvalid;
    C2 w{0.0, 0.0};
    if (!pauli::commute(xa, za, xb, zb)) {
      w = cmul(bval[a0 + ia], bval[b0 + ib]);
      w = pauli::apply_phase(cadd(w, w), pauli::phase_exponent(xa, za, xb, zb));
      key = ka ^ kb;
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
__global__ void combine_kernel(const int* __restrict__ off, int nseg, int n, const unsigned long long* __restrict__ key,
                               int pauli_q, int kbits, unsigned long long* __restrict__ ck) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int lo = 0, hi = nseg - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (off[mid] <= i) lo = mid;
      else hi = mid - 1;
    }
    const unsigned long long k = key[i];
    unsigned long long c;
    if (pauli_q > 0) {
      const bool inv = k == kInvalid;
      c = inv ? (1ull << kbits) : (key_x(k) | (key_z(k) << pauli_q));
    } else {
      c = k;
    }
    ck[i] = (static_cast<unsigned long long>(lo) << (kbits + 1)) | c;
  }
}
__global__ void split_kernel(const unsigned long long* __restrict__ ck, int n, int pauli_q, int kbits,
                             unsigned long long* __restrict__ ks, int* __restrict__ seg) {
  const unsigned long long kmask = (1ull << kbits) - 1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned long long c = ck[i];
    seg[i] = static_cast<int>(c >> (kbits + 1));
    if ((c >> kbits) & 1ull) {
      ks[i] = kInvalid;
    } else if (pauli_q > 0) {
      const unsigned long long k = c & kmask, qm = (1ull << pauli_q) - 1;
      ks[i] = pauli::pack(k & qm, k >> pauli_q);
    } else {
      ks[i] = c & kmask;
    }
  }
}

// first element of each (segment, key) run of the sorted keys
__global__ void heads_kernel(const unsigned long long* __restrict__ ks, const int* __restrict__ seg, int n,
                             int* __restrict__ flag) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    flag[i] = ks[i] != kInvalid && (i == 0 || seg[i] != seg[i - 1] || ks[i] != ks[i - 1]);
}

// from_terms accumulation: each run summed in input order from +0
__global__ void run_sum_kernel(const unsigned long long* __restrict__ ks, const unsigned* __restrict__ is,
                               const C2* __restrict__ val, const int* __restrict__ seg, const int* __restrict__ flag,
                               const int* __restrict__ pos, int n, unsigned long long* __restrict__ rkey,
                               C2* __restrict__ rval, double* __restrict__ rmag, int* __restrict__ rseg) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (!flag[i]) continue;
    const unsigned long long k = ks[i];
    C2 acc = pauli::slot(val[is[i]]);
    for (int j = i + 1; j < n && ks[j] == k && seg[j] == seg[i]; ++j) acc = cadd(acc, val[is[j]]);
    const int r = pos[i];
    rkey[r] = k;
    rval[r] = acc;
    rmag[r] = hypot(acc.re, acc.im);
    rseg[r] = seg[i];
  }
}

// out[p] = pos[off[p]] (positions before segment p), total past the end
__global__ void seg_positions_kernel(const int* __restrict__ off, int nseg, int n, const int* __restrict__ pos,
                                     int total, int* __restrict__ out) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p <= nseg; p += gridDim.x * blockDim.x)
    out[p] = (p < nseg && off[p] < n) ? pos[off[p]] : total;
}

// exclusive-scan total: pos[n-1] + flag[n-1]
__global__ void scan_total_kernel(const int* __restrict__ pos, const int* __restrict__ flag, int n,
                                  int* __restrict__ out) {
  *out = n > 0 ? pos[n - 1] + flag[n - 1] : 0;
}

__global__ void scan_total64_kernel(const long long* __restrict__ pos, const long long* __restrict__ cnt, int n,
                                    long long* __restrict__ out) {
  *out = n > 0 ? pos[n - 1] + cnt[n - 1] : 0;
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

__global__ void compact_kernel(const int* __restrict__ keep, const int* __restrict__ kpos, int n,
                               const unsigned long long* __restrict__ rkey, const C2* __restrict__ rval,
                               unsigned long long* __restrict__ okey, C2* __restrict__ oval) {
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

struct Index {
  unsigned long long* key;  // open-addressed slots (pauli::kEmpty = free)
  int* head;
  int* tail;
  int* count;
  uint64_t mask;
  int* e_l;  // entries, appended in accept order (so every list is ascending in l)
  C2* e_v;
  int* e_next;
};

__device__ __forceinline__ int index_find(const Index& ix, unsigned long long key) {
  for (uint64_t p = pauli::mix(key) & ix.mask;; p = (p + 1) & ix.mask) {
    const unsigned long long k = ix.key[p];
    if (k == pauli::kEmpty) return -1;
    if (k == key) return static_cast<int>(p);
  }
}

// Append the n terms (distinct keys) of accepted element l as entries e0...
__global__ void index_insert_kernel(Index ix, const unsigned long long* __restrict__ key, const C2* __restrict__ val,
                                    int n, int l, int e0) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int e = e0 + t;
    ix.e_l[e] = l;
    ix.e_v[e] = val[t];
    ix.e_next[e] = -1;
    const unsigned long long k = key[t];
    for (uint64_t p = pauli::mix(k) & ix.mask;; p = (p + 1) & ix.mask) {
      const unsigned long long prev = atomicCAS(&ix.key[p], pauli::kEmpty, k);
      if (prev == pauli::kEmpty) {
        ix.head[p] = e;
        ix.tail[p] = e;
        ix.count[p] = 1;
        break;
      }
      if (prev == k) {  // one thread per key in this launch
        ix.e_next[ix.tail[p]] = e;
        ix.tail[p] = e;
        ix.count[p] += 1;
        break;
      }
    }
  }
}

// move every occupied slot of `from` into `to` (lists unchanged)
__global__ void index_rehash_kernel(Index from, uint64_t from_slots, Index to) {
  for (uint64_t s = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; s < from_slots;
       s += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const unsigned long long k = from.key[s];
    if (k == pauli::kEmpty) continue;
    for (uint64_t p = pauli::mix(k) & to.mask;; p = (p + 1) & to.mask) {
      if (atomicCAS(&to.key[p], pauli::kEmpty, k) == pauli::kEmpty) {
        to.head[p] = from.head[s];
        to.tail[p] = from.tail[s];
        to.count[p] = from.count[s];
        break;
      }
    }
  }
}

__global__ void index_reset_kernel(Index ix, uint64_t slots) {
  for (uint64_t s = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; s < slots;
       s += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    ix.key[s] = pauli::kEmpty;
}

// overlap contributions of each term: one per basis element l < n_limit that
// holds the term's string
__global__ void beta_count_kernel(Index ix, const unsigned long long* __restrict__ key, int n, int n_limit,
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
__global__ void beta_fill_kernel(Index ix, const unsigned long long* __restrict__ key, const C2* __restrict__ val,
                                 int n, int n_limit, const long long* __restrict__ pos, unsigned long long* __restrict__ out_l,
                                 C2* __restrict__ out_v) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const int s = index_find(ix, key[t]);
    if (s < 0) continue;
    long long w = pos[t];
    for (int e = ix.head[s]; e >= 0 && ix.e_l[e] < n_limit; e = ix.e_next[e], ++w) {
      const C2 v = ix.e_v[e];
      out_l[w] = static_cast<unsigned long long>(ix.e_l[e]);
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
__global__ void chunk_base_kernel(const int* __restrict__ hoff, const int* __restrict__ broff, int nseg,
                                  Chunk* __restrict__ ch, long long* __restrict__ clen) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < nseg; p += gridDim.x * blockDim.x) {
    const int k = p + broff[p];
    ch[k] = {hoff[p + 1] - hoff[p], 0, hoff[p], {1.0, 0.0}};
    clen[k] = ch[k].len;
  }
}
__global__ void chunk_basis_kernel(const unsigned long long* __restrict__ bl, const C2* __restrict__ beta,
                                   const int* __restrict__ rseg, int nruns, const int64_t* __restrict__ voff,
                                   Chunk* __restrict__ ch, long long* __restrict__ clen) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nruns; r += gridDim.x * blockDim.x) {
    const int k = r + rseg[r] + 1;
    const int64_t l = static_cast<int64_t>(bl[r]);
    const C2 b = beta[r];
    const bool zero = b.re == 0.0 && b.im == 0.0;
    ch[k] = {zero ? 0 : static_cast<int>(voff[l + 1] - voff[l]), 1, voff[l], {-b.re, -b.im}};
    clen[k] = ch[k].len;
  }
}
// one block per chunk: coefficient = mult * term (base_coeff * t, coeffs[l] * t)
__global__ void chunk_fill_kernel(const Chunk* __restrict__ ch, const long long* __restrict__ cpos, int nchunks,
                                  const unsigned long long* __restrict__ hkey, const C2* __restrict__ hval,
                                  const unsigned long long* __restrict__ vkey, const C2* __restrict__ vval,
                                  unsigned long long* __restrict__ out_key, C2* __restrict__ out_val) {
  for (int k = blockIdx.x; k < nchunks; k += gridDim.x) {
    const Chunk c = ch[k];
    const unsigned long long* sk = (c.kind == 0 ? hkey : vkey) + c.src;
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
__global__ void append_scaled_kernel(const unsigned long long* __restrict__ key, const C2* __restrict__ val, int n,
                                     double rn, unsigned long long* __restrict__ okey, C2* __restrict__ oval) {
  const C2 s{__ddiv_rn(1.0, rn), 0.0};
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    okey[t] = key[t];
    oval[t] = cmul(val[t], s);
  }
}

} // namespace psum
} // namespace liecl_b200
