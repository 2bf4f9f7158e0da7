// K5: sparse Pauli-string frontier kernels (config 4), bit-exact.
//
// Every basis element of a closure over single Pauli strings is a single
// string (x, z) with one complex coefficient. A candidate bracket
// [V_l, V_m] (R:src/pauli.cpp:179-200) is null when the strings commute
// (symplectic parity, :68-71); otherwise its string is (x_l^x_m, z_l^z_m) with
// coefficient i^e * 2 c_l c_m (:50-59, apply_phase :26-33), normalised by its
// norm (:222-228). Independence against an orthonormal tuple of single
// strings (project_residual, R:src/closure.cpp:142-162 through the PauliSum
// branch of linear_combination, R:src/operator.cpp:164-181) reduces to
// membership: a string already in V cancels to (near) zero, a new one
// survives. Membership is an O(1) probe in a device hash set instead of the
// reference's O(|V|) term merge.
//
// Every floating-point operation of the reference is replayed in the same
// order with explicitly rounded intrinsics (no FMA contraction), so
// coefficients and residual norms match the reference bit for bit (the
// reference's own build has no FMA: x86-64 baseline ISA).
//
// Frontier batching: all pairs (l, m) with l < |V| at batch start are one
// batch. A pair whose string is already in V is rejected (it would be in the
// reference too: the span only grows); among new strings the first occurrence
// in cursor order is accepted and later duplicates are rejected as members of
// the then-current V -- exactly the sequential verdicts (strings within one
// row are distinct, so the reference's speculation never disagrees).
#pragma once

#include "common.cuh"

namespace liecl_b200 {
namespace pauli {

constexpr unsigned long long kEmpty = ~0ull;

struct C2 {
  double re, im;
};

// std::complex<double> a * b as the reference's build computes it.
__device__ __forceinline__ C2 cmul(C2 a, C2 b) {
  return {__dsub_rn(__dmul_rn(a.re, b.re), __dmul_rn(a.im, b.im)),
          __dadd_rn(__dmul_rn(a.re, b.im), __dmul_rn(a.im, b.re))};
}
__device__ __forceinline__ C2 cadd(C2 a, C2 b) { return {__dadd_rn(a.re, b.re), __dadd_rn(a.im, b.im)}; }
// value-initialised std::unordered_map slot += c (PauliSum::from_terms, R:src/pauli.cpp:93)
__device__ __forceinline__ C2 slot(C2 c) { return cadd({0.0, 0.0}, c); }
__device__ __forceinline__ bool is_zero(C2 c) { return c.re == 0.0 && c.im == 0.0; }
// sqrt(0 + std::norm(c)) (sum_norm of a one-term sum, R:src/pauli.cpp:222-228)
__device__ __forceinline__ double single_norm(C2 c) {
  return __dsqrt_rn(__dadd_rn(0.0, __dadd_rn(__dmul_rn(c.re, c.re), __dmul_rn(c.im, c.im))));
}
__device__ __forceinline__ C2 apply_phase(C2 c, unsigned e) {
  switch (e & 3u) {
  case 0: return c;
  case 1: return {-c.im, c.re};
  case 2: return {-c.re, -c.im};
  default: return {c.im, -c.re};
  }
}
__device__ __forceinline__ unsigned phase_exponent(uint64_t px, uint64_t pz, uint64_t qx, uint64_t qz) {
  const uint64_t rx = px ^ qx, rz = pz ^ qz;
  const int e = __popcll(px & pz) + __popcll(qx & qz) - __popcll(rx & rz) + 2 * __popcll(pz & qx);
  return static_cast<unsigned>(((e % 4) + 4) % 4);
}
__device__ __forceinline__ bool commute(uint64_t px, uint64_t pz, uint64_t qx, uint64_t qz) {
  return (__popcll((px & qz) ^ (pz & qx)) & 1) == 0;
}

__host__ __device__ __forceinline__ unsigned long long pack(uint64_t x, uint64_t z) {
  return static_cast<unsigned long long>(x) | (static_cast<unsigned long long>(z) << 32);
}
__device__ __forceinline__ uint64_t mix(unsigned long long k) {
  uint64_t h = k * 0x9E3779B97F4A7C15ull;
  h = (h ^ (h >> 30)) * 0xBF58476D1CE4E5B9ull;
  h = (h ^ (h >> 27)) * 0x94D049BB133111EBull;
  return h ^ (h >> 31);
}

// Open-addressed set of basis strings -> basis index. Keys are the whole
// (x, z) pair (128 bits), so strings on up to 64 qubits are keys
// (R:src/pauli.cpp:383-391; R:src/generators.cpp:32); slots are claimed with a
// 128-bit CAS. The empty marker (~0, ~0) is also the valid 64-qubit string
// Y^64; that one key lives in the extra slot keys[mask + 1] (tables hold
// mask + 2 slots), present when its value is not kNoVal.
constexpr long long kNoVal = 0x7fffffffffffffffll;

struct StringSet {
  ulonglong2* keys;  // (x, z)
  long long* vals;
  uint64_t mask;
};

__device__ __forceinline__ uint64_t mix2(uint64_t x, uint64_t z) { return mix(x ^ mix(z + 0x632BE59BD9B4E019ull)); }
__device__ __forceinline__ bool all_ones(uint64_t x, uint64_t z) { return (x & z) == ~0ull; }
__device__ __forceinline__ ulonglong2 cas128(ulonglong2* addr, ulonglong2 cmp, ulonglong2 val) {
  const unsigned __int128 c = (static_cast<unsigned __int128>(cmp.y) << 64) | cmp.x;
  const unsigned __int128 v = (static_cast<unsigned __int128>(val.y) << 64) | val.x;
  const unsigned __int128 r = atomicCAS(reinterpret_cast<unsigned __int128*>(addr), c, v);
  return make_ulonglong2(static_cast<unsigned long long>(r), static_cast<unsigned long long>(r >> 64));
}

// slot index of (x, z), or -1
__device__ __forceinline__ long long set_slot(const StringSet s, uint64_t x, uint64_t z) {
  if (all_ones(x, z)) return s.vals[s.mask + 1] == kNoVal ? -1 : static_cast<long long>(s.mask + 1);
  for (uint64_t p = mix2(x, z) & s.mask;; p = (p + 1) & s.mask) {
    const ulonglong2 k = s.keys[p];
    if (k.x == x && k.y == z) return static_cast<long long>(p);
    if (k.x == ~0ull && k.y == ~0ull) return -1;
  }
}
__device__ __forceinline__ long long set_find(const StringSet s, uint64_t x, uint64_t z) {
  const long long p = set_slot(s, x, z);
  return p < 0 ? -1 : s.vals[p];
}
__device__ __forceinline__ void set_insert(StringSet s, uint64_t x, uint64_t z, long long val) {
  if (all_ones(x, z)) {
    s.vals[s.mask + 1] = val;
    return;
  }
  const ulonglong2 key = make_ulonglong2(x, z), empty = make_ulonglong2(~0ull, ~0ull);
  for (uint64_t p = mix2(x, z) & s.mask;; p = (p + 1) & s.mask) {
    const ulonglong2 prev = cas128(&s.keys[p], empty, key);
    if ((prev.x == ~0ull && prev.y == ~0ull) || (prev.x == x && prev.y == z)) {
      s.vals[p] = val;
      return;
    }
  }
}
// Batch-local first-occurrence table: key -> min candidate position.
__device__ __forceinline__ void first_insert(StringSet s, uint64_t x, uint64_t z, long long pos) {
  if (all_ones(x, z)) {
    atomicMin(&s.vals[s.mask + 1], pos);
    return;
  }
  const ulonglong2 key = make_ulonglong2(x, z), empty = make_ulonglong2(~0ull, ~0ull);
  for (uint64_t p = mix2(x, z) & s.mask;; p = (p + 1) & s.mask) {
    const ulonglong2 prev = cas128(&s.keys[p], empty, key);
    if ((prev.x == ~0ull && prev.y == ~0ull) || (prev.x == x && prev.y == z)) {
      atomicMin(&s.vals[p], pos);
      return;
    }
  }
}

// One linear_combination pass (R:src/operator.cpp:164-181 + from_terms) of a
// one-term base (string key, coefficient c) against V; `v` is the basis
// coefficient of the same string when it is a member. Returns false for the
// empty sum (all terms cancelled / dropped).
__device__ __forceinline__ bool project_pass(bool member, C2 v, C2 c, C2& out) {
  C2 acc = slot(cmul({1.0, 0.0}, c));
  if (member) {
    const C2 beta = slot(cmul({v.re, -v.im}, c));  // sum_inner_product: 0 + conj(v) * c
    acc = cadd(acc, cmul({-beta.re, -beta.im}, v));
  }
  if (is_zero(acc)) return false;  // |acc| > 1e-14 |acc| <=> acc != 0
  out = acc;
  return true;
}

// OrthonormStrategy::check of a one-term candidate (R:src/closure.cpp:276-286).
__device__ __forceinline__ double check(bool basis_empty, bool member, C2 v, C2 h, double tol, bool& indep,
                                        C2& unit) {
  C2 r = h;
  bool alive = true;
  if (!basis_empty) {
    alive = project_pass(member, v, h, r);
    if (alive) alive = project_pass(member, v, r, r);
  }
  const double rn = alive ? single_norm(r) : 0.0;
  indep = rn > tol;
  if (indep) unit = cmul(r, {__ddiv_rn(1.0, rn), 0.0});
  return rn;
}

enum Verdict : int { kNull = 0, kMember = 1, kNew = 2, kAccepted = 3, kDuplicate = 4 };

struct CandidateOut {
  uint64_t* x;
  uint64_t* z;
  C2* hunit;   // normalised candidate (Alg. 3 originals)
  C2* unit;    // residual unit (appended to V when accepted)
  double* rn;  // residual norm of the verdict
  int* verdict;
  int* flags;  // bit0: borderline residual, bit1: member residual above tol (unsupported)
};

// Candidate stage. mode 0: generators gx/gz/gc [0, count); mode 1: cursor
// pairs [g0, g0 + count) over the commutator basis (vx, vz, cb).
__global__ void candidates_kernel(int mode, int64_t g0, int count, const uint64_t* __restrict__ gx,
                                  const uint64_t* __restrict__ gz, const C2* __restrict__ gc,
                                  const uint64_t* __restrict__ vx, const uint64_t* __restrict__ vz,
                                  const C2* __restrict__ vc, const C2* __restrict__ cb, long long nv,
                                  StringSet vset, StringSet first, double tol, CandidateOut out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= count) return;
  uint64_t x, z;
  C2 h;
  bool nul;
  if (mode == 0) {
    // generator loop (R:src/closure.cpp:378-388): from_terms stored 0 + c
    x = gx[j];
    z = gz[j];
    const C2 g = slot(gc[j]);
    const double gn = is_zero(g) ? 0.0 : single_norm(g);
    nul = !(gn > tol);
    h = nul ? C2{0.0, 0.0} : cmul(g, {__ddiv_rn(1.0, gn), 0.0});
    if (nul) out.rn[j] = gn;
  } else {
    int64_t l, m;
    pair_from_index(g0 + j, l, m);
    const uint64_t px = vx[l], pz = vz[l], qx = vx[m], qz = vz[m];
    x = px ^ qx;
    z = pz ^ qz;
    nul = commute(px, pz, qx, qz);
    if (!nul) {
      C2 w = cmul(cb[l], cb[m]);
      w = slot(apply_phase(cadd(w, w), phase_exponent(px, pz, qx, qz)));
      const double hn = is_zero(w) ? 0.0 : single_norm(w);
      nul = !(hn > tol);
      if (!nul) h = cmul(w, {__ddiv_rn(1.0, hn), 0.0});
    }
    if (nul) out.rn[j] = 0.0;
  }
  out.x[j] = x;
  out.z[j] = z;
  int flags = 0;
  if (nul) {
    out.verdict[j] = kNull;
    out.flags[j] = 0;
    return;
  }
  out.hunit[j] = h;
  const long long idx = nv > 0 ? set_find(vset, x, z) : -1;
  bool indep;
  C2 unit = {0.0, 0.0};
  const double rn = check(nv == 0, idx >= 0, idx >= 0 ? vc[idx] : C2{0.0, 0.0}, h, tol, indep, unit);
  out.rn[j] = rn;
  out.unit[j] = unit;
  if (rn > 0.0 && rn >= tol / 10.0 && rn <= tol * 10.0) flags |= 1;
  if (idx >= 0) {
    if (indep) flags |= 2;
    out.verdict[j] = kMember;
  } else {
    out.verdict[j] = indep ? kNew : kMember;  // kMember here: new string but residual <= tol
    if (indep) first_insert(first, x, z, j);
  }
  out.flags[j] = flags;
}

// First occurrence among new strings wins; later duplicates are checked
// against the winner (a member of the then-current V).
__global__ void resolve_kernel(int count, StringSet first, double tol, CandidateOut out,
                               int* __restrict__ accept_flag) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= count) return;
  int acc = 0;
  if (out.verdict[j] == kNew) {
    const long long win = set_find(first, out.x[j], out.z[j]);
    if (win == j) {
      out.verdict[j] = kAccepted;
      acc = 1;
    } else {
      bool indep;
      C2 unit;
      const double rn = check(false, true, out.unit[win], out.hunit[j], tol, indep, unit);
      out.rn[j] = rn;
      out.verdict[j] = kDuplicate;
      int f = 0;
      if (rn > 0.0 && rn >= tol / 10.0 && rn <= tol * 10.0) f |= 1;
      if (indep) f |= 2;
      out.flags[j] = f;
    }
  }
  accept_flag[j] = acc;
}

// Append accepted candidates at nv + rank (rank = exclusive scan of accept_flag).
__global__ void append_kernel(int count, const int* __restrict__ accept_flag, const int* __restrict__ rank,
                              long long nv, CandidateOut in, uint64_t* __restrict__ vx, uint64_t* __restrict__ vz,
                              C2* __restrict__ vc, C2* __restrict__ oc, StringSet vset) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= count || !accept_flag[j]) return;
  const long long p = nv + rank[j];
  vx[p] = in.x[j];
  vz[p] = in.z[j];
  vc[p] = in.unit[j];
  if (oc) oc[p] = in.hunit[j];
  set_insert(vset, in.x[j], in.z[j], p);
}

// ---- persistent frontier: the whole cursor loop in one CTA ---------------
//
// While the frontier (available pairs not yet visited) is narrow, one CTA of
// 1024 threads runs run_engine's loop (R:src/closure.cpp:378-460) with no host
// round trip: the generator loop on one thread (sequential, as the
// reference), then chunks of up to 1024 consecutive cursor pairs. A chunk is
// checked against V as it stands at the chunk start; the first new
// occurrence of a string in the chunk is accepted and later ones are checked
// against it (resolve_kernel's rule); accepts are appended in cursor order
// (ballot scan) and inserted into the string set before the next chunk. The
// launch stops when the loop is done, the frontier outgrows `wide` (the
// multi-CTA batches take over), the log arrays fill up, or the basis buffers
// are full (the host grows them and relaunches; the chunk is redone).
enum FrontierStatus : int { kDone = 0, kWide = 1, kCapacity = 2, kLogFull = 3, kGrow = 4 };

struct FrontierState {
  long long n;  // basis size
  long long g;  // next cursor pair
  unsigned long long checks, border, bad, chunks;
  int status;
  int pad;
};

constexpr int kFrontierThreads = 1024;
constexpr int kFirstSlots = 2048;

__device__ __forceinline__ int flags_of(double rn, double tol) {
  return (rn > 0.0 && rn >= tol / 10.0 && rn <= tol * 10.0) ? 1 : 0;
}

// basis arrays are written and re-read by this CTA: plain (coherent) loads
__global__ void __launch_bounds__(kFrontierThreads, 1)
frontier_kernel(int ngens, const uint64_t* __restrict__ gx, const uint64_t* __restrict__ gz,
                const C2* __restrict__ gc, uint64_t* vx, uint64_t* vz, C2* vc, C2* oc, StringSet vset,
                long long vcap, long long cap, double tol, CandidateOut out, long long out_cap, long long wide,
                FrontierState* st) {
  __shared__ int s_slot[kFirstSlots];
  __shared__ int s_min[kFirstSlots];
  __shared__ uint64_t s_x[kFrontierThreads], s_z[kFrontierThreads];
  __shared__ int s_warp[kFrontierThreads / 32];
  __shared__ long long s_n, s_g;
  __shared__ unsigned long long s_cnt[4];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const C2* cb = oc ? oc : vc;  // Alg. 3 brackets the originals
  const long long g_launch = st->g;
  int status = kDone;

  if (tid == 0) {
    long long n = st->n;
    unsigned long long checks = 0, border = 0, bad = 0;
    // generator loop (R:src/closure.cpp:378-403), appended as accepted
    for (int j = 0; j < ngens; ++j) {
      const uint64_t x = gx[j], z = gz[j];
      out.x[j] = x;
      out.z[j] = z;
      out.flags[j] = 0;
      const C2 g = slot(gc[j]);
      const double gn = is_zero(g) ? 0.0 : single_norm(g);
      if (!(gn > tol)) {
        out.verdict[j] = kNull;
        out.rn[j] = gn;
        continue;
      }
      ++checks;
      const C2 h = cmul(g, {__ddiv_rn(1.0, gn), 0.0});
      out.hunit[j] = h;
      const long long idx = n > 0 ? set_find(vset, x, z) : -1;
      bool indep;
      C2 unit = {0.0, 0.0};
      const double rn = check(n == 0, idx >= 0, idx >= 0 ? vc[idx] : C2{0.0, 0.0}, h, tol, indep, unit);
      out.rn[j] = rn;
      out.unit[j] = unit;
      const int f = flags_of(rn, tol) | ((idx >= 0 && indep) ? 2 : 0);
      out.flags[j] = f;
      border += f & 1;
      bad += (f >> 1) & 1;
      if (indep && idx < 0) {
        if (n + 1 > cap) {
          status = kCapacity;
          break;
        }
        out.verdict[j] = kAccepted;
        vx[n] = x;
        vz[n] = z;
        vc[n] = unit;
        if (oc) oc[n] = h;
        set_insert(vset, x, z, n);
        ++n;
      } else {
        out.verdict[j] = kMember;
      }
    }
    s_n = n;
    s_g = g_launch;
    s_cnt[0] = checks;
    s_cnt[1] = border;
    s_cnt[2] = bad;
    s_cnt[3] = 0;
    s_warp[0] = status;
  }
  __syncthreads();
  status = s_warp[0];
  unsigned long long checks = 0, border = 0, bad = 0, chunks = 0;  // thread 0's running totals
  const long long base = ngens;
  while (status == kDone) {
    const long long n = s_n, g = s_g;
    const long long avail = n * (n - 1) / 2;
    if (g >= avail) break;
    if (avail - g > wide) { status = kWide; break; }
    const int cnt = static_cast<int>(avail - g < kFrontierThreads ? avail - g : kFrontierThreads);
    const long long o0 = base + (g - g_launch);
    if (o0 + cnt > out_cap) { status = kLogFull; break; }
    for (int i = tid; i < kFirstSlots; i += kFrontierThreads) {
      s_slot[i] = -1;
      s_min[i] = kFrontierThreads;
    }
    __syncthreads();
    const int j = tid;
    int verdict = kNull, flags = 0, myslot = -1;
    uint64_t x = 0, z = 0;
    C2 h = {0.0, 0.0}, unit = {0.0, 0.0};
    if (j < cnt) {
      int64_t l, m;
      pair_from_index(g + j, l, m);
      const uint64_t px = vx[l], pz = vz[l], qx = vx[m], qz = vz[m];
      x = px ^ qx;
      z = pz ^ qz;
      bool nul = commute(px, pz, qx, qz);
      if (!nul) {
        C2 w = cmul(cb[l], cb[m]);
        w = slot(apply_phase(cadd(w, w), phase_exponent(px, pz, qx, qz)));
        const double hn = is_zero(w) ? 0.0 : single_norm(w);
        nul = !(hn > tol);
        if (!nul) h = cmul(w, {__ddiv_rn(1.0, hn), 0.0});
      }
      out.x[o0 + j] = x;
      out.z[o0 + j] = z;
      if (nul) {
        out.rn[o0 + j] = 0.0;
      } else {
        out.hunit[o0 + j] = h;
        const long long idx = set_find(vset, x, z);  // n >= 2 here
        bool indep;
        const double rn = check(false, idx >= 0, idx >= 0 ? vc[idx] : C2{0.0, 0.0}, h, tol, indep, unit);
        out.rn[o0 + j] = rn;
        out.unit[o0 + j] = unit;
        flags = flags_of(rn, tol);
        if (idx >= 0) {
          if (indep) flags |= 2;
          verdict = kMember;
        } else if (indep) {
          verdict = kNew;
          s_x[j] = x;
          s_z[j] = z;
          __threadfence_block();
          for (int p = static_cast<int>(mix2(x, z) & (kFirstSlots - 1));; p = (p + 1) & (kFirstSlots - 1)) {
            const int prev = atomicCAS(&s_slot[p], -1, j);
            __threadfence_block();  // pairs with the writer's fence: s_x/s_z[prev] are visible
            if (prev == -1 || (s_x[prev] == x && s_z[prev] == z)) {
              atomicMin(&s_min[p], j);
              myslot = p;
              break;
            }
          }
        } else {
          verdict = kMember;  // new string, residual <= tol
        }
      }
    }
    __syncthreads();
    bool acc = false;
    if (verdict == kNew) {
      const int win = s_min[myslot];
      if (win == j) {
        acc = true;
        verdict = kAccepted;
      } else {
        bool indep;
        C2 u2;
        const double rn = check(false, true, out.unit[o0 + win], h, tol, indep, u2);
        out.rn[o0 + j] = rn;
        verdict = kDuplicate;
        flags = flags_of(rn, tol) | (indep ? 2 : 0);
      }
    }
    if (j < cnt) {
      out.verdict[o0 + j] = verdict;
      out.flags[o0 + j] = flags;
    }
    // accept ranks in cursor order
    const unsigned ball = __ballot_sync(0xffffffffu, acc);
    if (lane == 0) s_warp[warp] = __popc(ball);
    const int c_checks = __syncthreads_count(j < cnt && verdict != kNull);
    const int c_border = __syncthreads_count(flags & 1);
    const int c_bad = __syncthreads_count((flags >> 1) & 1);
    int before = 0, total = 0;
#pragma unroll 4
    for (int w = 0; w < kFrontierThreads / 32; ++w) {
      const int c = s_warp[w];
      before += w < warp ? c : 0;
      total += c;
    }
    if (n + total > cap) {
      if (tid == 0) bad += c_bad;
      status = kCapacity;
      break;
    }
    if (n + total > vcap) { status = kGrow; break; }
    if (acc) {
      const long long p = n + before + __popc(ball & ((1u << lane) - 1u));
      vx[p] = x;
      vz[p] = z;
      vc[p] = unit;
      if (oc) oc[p] = h;
      set_insert(vset, x, z, p);
    }
    if (tid == 0) {
      checks += c_checks;
      border += c_border;
      bad += c_bad;
      ++chunks;
      s_n = n + total;
      s_g = g + cnt;
    }
    __syncthreads();
  }
  if (tid == 0) {
    st->n = s_n;
    st->g = s_g;
    st->checks = s_cnt[0] + checks;
    st->border = s_cnt[1] + border;
    st->bad = s_cnt[2] + bad;
    st->chunks = chunks;
    st->status = status;
  }
}

// ---- exclusive scan of accept flags (the wide batches' append ranks) -------
// Three launches: per-1024 block scans with their totals, one block scanning
// the (<= 4096) totals, block offsets added back. Batches hold <= 4M pairs.
constexpr int kScanBlock = 1024;
__device__ __forceinline__ int block_exclusive_scan(int v, int* s_warp, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < static_cast<int>(blockDim.x >> 5) ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    s_warp[lane] = w;  // inclusive prefix of warp totals
  }
  __syncthreads();
  total = s_warp[(blockDim.x >> 5) - 1];
  return (warp > 0 ? s_warp[warp - 1] : 0) + x - v;
}
__global__ void __launch_bounds__(kScanBlock) scan_blocks_kernel(const int* __restrict__ in, int n,
                                                                 int* __restrict__ out, int* __restrict__ sums) {
  __shared__ int s_warp[32];
  const int i = blockIdx.x * kScanBlock + threadIdx.x;
  int total;
  const int e = block_exclusive_scan(i < n ? in[i] : 0, s_warp, total);
  if (i < n) out[i] = e;
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}
// one block of kScanBlock threads: exclusive scan of nb <= 4 kScanBlock totals, grand total at sums[nb]
__global__ void __launch_bounds__(kScanBlock) scan_sums_kernel(int* __restrict__ sums, int nb) {
  __shared__ int s_warp[32];
  int v[4], t = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int i = threadIdx.x * 4 + k;
    v[k] = i < nb ? sums[i] : 0;
    t += v[k];
  }
  int total;
  int run = block_exclusive_scan(t, s_warp, total);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int i = threadIdx.x * 4 + k;
    if (i < nb) sums[i] = run;
    run += v[k];
  }
  if (threadIdx.x == 0) sums[nb] = total;
}
__global__ void scan_add_kernel(int* __restrict__ out, int n, const int* __restrict__ sums) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] += sums[i / kScanBlock];
}

// n = mask + 2 slots
__global__ void reset_table_kernel(StringSet s, uint64_t n) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    s.keys[i] = make_ulonglong2(~0ull, ~0ull);
    s.vals[i] = kNoVal;
  }
}

} // namespace pauli
} // namespace liecl_b200
