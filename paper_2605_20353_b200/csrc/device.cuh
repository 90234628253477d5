// device.cuh -- device-side building blocks of the sample kernels:
// Philox4x32-10 counter RNG (reading R11), index maps, COO record fetch and the
// hash-set membership probe, and the three losses (reading R3).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "gcp_internal.h"

namespace gcp {

// ---- Philox4x32-10 ---------------------------------------------------------
// Ten rounds of (c0,c1,c2,c3) -> (hi(M1 c2)^c1^k0, lo(M1 c2), hi(M0 c0)^c3^k1,
// lo(M0 c0)); key bumped by the Weyl constants between rounds.
struct U64x2 { uint64_t w0, w1; };

__device__ __forceinline__ U64x2 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                        uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
        const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    U64x2 o;
    o.w0 = (uint64_t)c0 | ((uint64_t)c1 << 32);
    o.w1 = (uint64_t)c2 | ((uint64_t)c3 << 32);
    return o;
}

// floor(W * n / 2^64): an exact integer map of a uniform 64-bit word onto [0, n).
__device__ __forceinline__ uint64_t range_map(uint64_t W, uint64_t n) { return __umul64hi(W, n); }

// Philox iteration word: inside a replayed epoch graph the replay's first
// iteration (device memory) plus this launch's offset, else the launch argument.
__device__ __forceinline__ uint32_t iter_word(const SampleArgs& a) { return a.it_dev ? *a.it_dev + a.it : a.it; }

// ---- hashing ------------------------------------------------------------------
__device__ __host__ __forceinline__ uint64_t mix64(uint64_t z) {   // splitmix64 finaliser
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t hash_key(uint64_t lo, uint64_t hi) { return mix64(lo ^ mix64(hi + 0x9E3779B97F4A7C15ull)); }

constexpr uint64_t kEmpty = ~0ull;

// Blocked Bloom filter in front of the exact zero test: a key owns one 32-byte
// sector (4 u64 words) and sets one bit in each word.  Sized to stay in L2
// (ingest.cu); a zero candidate reads its sector instead of a DRAM bucket and
// runs the exact test (hash probe or row f4's O(log N) search) only on
// "maybe".  No false negatives.  In front of the sorted search it is used
// from 4 bits per key (c2: 5.4 bits, ~8% false positives, f4 K2 3x faster); in
// front of the hash only from 12 bits per key (< 1% false positives), since a
// "maybe" stalls its warp on a synchronous probe (profiles/r01_summary.md).
__device__ __forceinline__ uint64_t filter_hash(uint64_t klo, uint64_t khi) {
    return mix64(hash_key(klo, khi) ^ 0x5851F42D4C957F2Dull);
}
__device__ __forceinline__ bool filter_maybe(const uint4& w0, const uint4& w1, uint64_t fh) {
    const uint64_t q0 = ((uint64_t)w0.y << 32) | w0.x, q1 = ((uint64_t)w0.w << 32) | w0.z;
    const uint64_t q2 = ((uint64_t)w1.y << 32) | w1.x, q3 = ((uint64_t)w1.w << 32) | w1.z;
    return ((q0 >> ((fh >> 32) & 63)) & (q1 >> ((fh >> 38) & 63)) & (q2 >> ((fh >> 44) & 63)) &
            (q3 >> ((fh >> 50) & 63)) & 1ull) != 0;
}

// Bucketised linear probing: a key hashes to a 32-byte bucket (4 u64 slots or
// 2 u128 slots); insertion and lookup scan slots from the bucket start, so an
// empty slot proves absence.  One 32-B sector per probe at load <= 0.5.
__device__ __forceinline__ bool set_contains64(const uint64_t* __restrict__ h, uint64_t mask, uint64_t key) {
    uint64_t s = (hash_key(key, 0) & mask) & ~3ull;
    for (;;) {
        const ulonglong2 a = __ldg(reinterpret_cast<const ulonglong2*>(h + s));
        const ulonglong2 b = __ldg(reinterpret_cast<const ulonglong2*>(h + s + 2));
        if (a.x == key || a.y == key || b.x == key || b.y == key) return true;
        if (a.x == kEmpty || a.y == kEmpty || b.x == kEmpty || b.y == kEmpty) return false;
        s = (s + 4) & mask;
    }
}
__device__ __forceinline__ bool set_contains128(const uint64_t* __restrict__ h, uint64_t mask,
                                                uint64_t klo, uint64_t khi) {
    // slots are (lo, hi) pairs: slot index s occupies h[2s], h[2s+1]
    uint64_t s = (hash_key(klo, khi) & mask) & ~1ull;
    for (;;) {
        const ulonglong2 a = __ldg(reinterpret_cast<const ulonglong2*>(h + 2 * s));
        const ulonglong2 b = __ldg(reinterpret_cast<const ulonglong2*>(h + 2 * s + 2));
        if ((a.x == klo && a.y == khi) || (b.x == klo && b.y == khi)) return true;
        if ((a.x == kEmpty && a.y == kEmpty) || (b.x == kEmpty && b.y == kEmpty)) return false;
        s = (s + 2) & mask;
    }
}

// ---- losses (reading R3), in the kernel precision T -----------------------------
template <typename T> __device__ __forceinline__ T d_log(T x);
template <> __device__ __forceinline__ float d_log<float>(float x) { return logf(x); }
template <> __device__ __forceinline__ double d_log<double>(double x) { return log(x); }
template <typename T> __device__ __forceinline__ T d_log1p(T x);
template <> __device__ __forceinline__ float d_log1p<float>(float x) { return log1pf(x); }
template <> __device__ __forceinline__ double d_log1p<double>(double x) { return log1p(x); }
template <typename T> __device__ __forceinline__ T d_exp(T x);
template <> __device__ __forceinline__ float d_exp<float>(float x) { return expf(x); }
template <> __device__ __forceinline__ double d_exp<double>(double x) { return exp(x); }

template <typename T> __device__ __forceinline__ T sigmoid(T m) {
    if (m >= T(0)) return T(1) / (T(1) + d_exp<T>(-m));
    const T e = d_exp<T>(m);
    return e / (T(1) + e);
}

// df/dm(x, m)
template <typename T> __device__ __forceinline__ T loss_df(int loss, T x, T m) {
    if (loss == GCP_LOSS_GAUSSIAN) return T(2) * (m - x);
    if (loss == GCP_LOSS_POISSON) return T(1) - x / (m + T(1e-10));
    return sigmoid<T>(m) - x;
}
// f(x, m)
template <typename T> __device__ __forceinline__ T loss_f(int loss, T x, T m) {
    if (loss == GCP_LOSS_GAUSSIAN) { const T e = x - m; return e * e; }
    if (loss == GCP_LOSS_POISSON) return m - x * d_log<T>(m + T(1e-10));
    const T sp = (m > T(0) ? m : T(0)) + d_log1p<T>(d_exp<T>(-fabs(m)));
    return sp - x * m;
}

// ---- one sample: index generation, record fetch / probe (rows a1, a2) ------------
template <typename T, int D>
struct Sample {
    uint32_t c[D];   // block-local coordinates
    T x;             // data value (0 for zero samples)
    int64_t j;       // canonical nonzero index, -1 for zeros
    int attempts;
    bool nz;
};

template <typename T> __device__ __forceinline__ T load_val(const uint32_t* r);
template <> __device__ __forceinline__ float load_val<float>(const uint32_t* r) { return __uint_as_float(r[0]); }
template <> __device__ __forceinline__ double load_val<double>(const uint32_t* r) {
    return __hiloint2double((int)r[1], (int)r[0]);
}

// A sample whose one dependent DRAM access (the COO record of a nonzero slot,
// or the first hash bucket of a zero candidate) has been issued but not yet
// consumed.  Splitting draw into issue + resolve lets the kernel keep the next
// chunk's random DRAM reads in flight while it works on the current chunk.
template <int D>
struct Pending {
    uint4 w0, w1;        // record words / bucket words as loaded
    uint32_t c[D];       // zero candidate (attempt 0)
    uint32_t slot;       // local slot within the stratum
    int state;           // 0 invalid, 1 nonzero, 2 zero (bucket loaded), 3 zero (no probe needed),
                         // 4 zero (sorted search at resolve), 5 zero (filter sector loaded)
    uint32_t j;          // nonzero index (low 32 bits; high bits recomputed if N >= 2^32)
};

template <int D>
__device__ __forceinline__ void zero_candidate(const SampleArgs& a, uint32_t zs, uint32_t att, uint32_t (&c)[D]) {
    const uint32_t k0 = (uint32_t)a.seed, k1 = (uint32_t)(a.seed >> 32);
#pragma unroll
    for (int g = 0; g < (D + 1) / 2; ++g) {
        const U64x2 w = philox(zs, a.rank, (a.kind_z << 28) | (att << 4) | (uint32_t)g, iter_word(a), k0, k1);
        c[2 * g] = (uint32_t)range_map(w.w0, a.bdim[2 * g]);
        GCP_CHECK(c[2 * g] < a.bdim[2 * g], "zero candidate coordinate", c[2 * g], a.bdim[2 * g]);
        if (2 * g + 1 < D) c[2 * g + 1] = (uint32_t)range_map(w.w1, a.bdim[2 * g + 1]);
    }
}

// first bucket (32 B) of the probe sequence of candidate c, as a word offset into the table
template <int D>
__device__ __forceinline__ uint64_t first_bucket(const SampleArgs& a, const uint32_t (&c)[D], uint64_t& klo,
                                                 uint64_t& khi) {
    if (!a.key128) {
        uint64_t key = c[0];
#pragma unroll
        for (int k = 1; k < D; ++k) key = key * a.bdim[k] + c[k];
        klo = key;
        khi = 0;
        return (hash_key(key, 0) & a.hash_mask) & ~3ull;
    }
    unsigned __int128 key = c[0];
#pragma unroll
    for (int k = 1; k < D; ++k) key = key * a.bdim[k] + c[k];
    klo = (uint64_t)key;
    khi = (uint64_t)(key >> 64);
    return 2 * ((hash_key(klo, khi) & a.hash_mask) & ~1ull);
}

// 16-B read of a line used once (record, hash bucket): with l2_first an L2
// evict_first cache policy so it does not displace the reused factor rows
__device__ __forceinline__ uint4 ldg_once(const uint4* p, int l2_first) {
    if (!l2_first) return __ldg(p);
    uint4 v;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}

template <typename T, int D>
__device__ __forceinline__ Pending<D> issue_sample(const SampleArgs& a, int64_t s) {
    Pending<D> P;
    P.state = 0;
    if (s >= a.p + a.q) return P;
    const uint32_t k0 = (uint32_t)a.seed, k1 = (uint32_t)(a.seed >> 32);
    constexpr int VW = (int)(sizeof(T) / 4);
    if (s < a.p) {
        // nonzero slot: j uniform over [0, N) with replacement
        const U64x2 w = philox((uint32_t)s, a.rank, a.kind_nz << 28, iter_word(a), k0, k1);
        const uint64_t j = range_map(w.w0, (uint64_t)a.N);
        GCP_CHECK(j < (uint64_t)a.N || a.rec_words == 0, "record index >= N", j, a.N);
        const uint4* r = reinterpret_cast<const uint4*>(a.rec + j * a.rec_words);
        P.w0 = ldg_once(r, a.l2_first);
        if (VW + D > 4) P.w1 = ldg_once(r + 1, a.l2_first);
        P.slot = (uint32_t)s;
        P.j = (uint32_t)j;
        P.state = 1;
        return P;
    }
    // zero slot, attempt 0: draw d indices and issue the first probe
    P.slot = (uint32_t)(s - a.p);
    zero_candidate<D>(a, P.slot, 0u, P.c);
    if (!a.stratified) {
        P.state = 3;
        return P;
    }
    uint64_t klo, khi;
    const uint64_t b = first_bucket<D>(a, P.c, klo, khi);
    if (a.filter) {          // the filter sector (L2); the exact test only on "maybe"
        const uint4* f = reinterpret_cast<const uint4*>(a.filter + 4 * (filter_hash(klo, khi) & a.filter_mask));
        P.w0 = __ldg(f);
        P.w1 = __ldg(f + 1);
        P.state = 5;
        return P;
    }
    if (a.member_sorted) {   // row f4: O(log N) search of the sorted keys at resolve time
        P.state = 4;
        return P;
    }
    GCP_CHECK(b + 4 <= (a.hash_mask + 1) * (a.key128 ? 2 : 1), "hash bucket past the table", b, a.hash_mask);
    const uint4* h = reinterpret_cast<const uint4*>(a.hash + b);
    P.w0 = ldg_once(h, a.l2_first);
    P.w1 = ldg_once(h + 1, a.l2_first);
    P.state = 2;
    return P;
}

// Row f4: lower-bound binary search of the canonical (sorted) key
// array; u128 keys are stored as (lo, hi) pairs.
__device__ __forceinline__ bool sorted_contains(const SampleArgs& a, uint64_t klo, uint64_t khi) {
    int64_t lo = 0, hi = a.N;   // search [lo, hi)
    while (lo < hi) {
        const int64_t mid = lo + ((hi - lo) >> 1);
        uint64_t mlo, mhi = 0;
        if (a.key128) {
            const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(a.keys) + mid);
            mlo = v.x;
            mhi = v.y;
        } else {
            mlo = __ldg(a.keys + mid);
        }
        if (mhi == khi && mlo == klo) return true;
        if (mhi < khi || (mhi == khi && mlo < klo)) lo = mid + 1;
        else hi = mid;
    }
    return false;
}

// 0 absent, 1 present, 2 undecided (bucket full of other keys: continue probing)
__device__ __forceinline__ int bucket_verdict(const SampleArgs& a, const uint4& w0, const uint4& w1, uint64_t klo,
                                              uint64_t khi) {
    const uint64_t s0 = ((uint64_t)w0.y << 32) | w0.x, s1 = ((uint64_t)w0.w << 32) | w0.z;
    const uint64_t s2 = ((uint64_t)w1.y << 32) | w1.x, s3 = ((uint64_t)w1.w << 32) | w1.z;
    if (!a.key128) {
        if (s0 == klo || s1 == klo || s2 == klo || s3 == klo) return 1;
        if (s0 == kEmpty || s1 == kEmpty || s2 == kEmpty || s3 == kEmpty) return 0;
        return 2;
    }
    if ((s0 == klo && s1 == khi) || (s2 == klo && s3 == khi)) return 1;
    if ((s0 == kEmpty && s1 == kEmpty) || (s2 == kEmpty && s3 == kEmpty)) return 0;
    return 2;
}

__device__ __forceinline__ bool probe_from(const SampleArgs& a, uint64_t klo, uint64_t khi) {
    if (a.member_sorted) return sorted_contains(a, klo, khi);
    return a.key128 ? set_contains128(a.hash, a.hash_mask, klo, khi) : set_contains64(a.hash, a.hash_mask, klo);
}

template <typename T, int D>
__device__ __forceinline__ Sample<T, D> resolve_sample(const SampleArgs& a, const Pending<D>& P) {
    Sample<T, D> o;
    constexpr int VW = (int)(sizeof(T) / 4);
    if (P.state == 1) {
        const uint32_t w8[8] = {P.w0.x, P.w0.y, P.w0.z, P.w0.w, P.w1.x, P.w1.y, P.w1.z, P.w1.w};
        o.x = load_val<T>(w8);
#pragma unroll
        for (int k = 0; k < D; ++k) o.c[k] = w8[(VW + k) & 7];
        uint64_t j = P.j;
        if ((uint64_t)a.N > 0xFFFFFFFFull) {
            const U64x2 w = philox(P.slot, a.rank, a.kind_nz << 28, iter_word(a), (uint32_t)a.seed, (uint32_t)(a.seed >> 32));
            j = range_map(w.w0, (uint64_t)a.N);
        }
        o.j = (int64_t)j;
        o.attempts = 1;
        o.nz = true;
        return o;
    }
    o.x = T(0);
    o.j = -1;
    o.nz = false;
    o.attempts = 1;
#pragma unroll
    for (int k = 0; k < D; ++k) o.c[k] = P.c[k];
    if (P.state != 2 && P.state != 4 && P.state != 5) return o;
    // zero candidate: decide attempt 0 from the prefetched bucket (or the filter
    // sector + sorted search); rejected candidates redraw all d indices
    // -- rare, inline
    uint64_t klo, khi;
    first_bucket<D>(a, o.c, klo, khi);
    bool present;
    if (P.state == 5) {
        present = filter_maybe(P.w0, P.w1, filter_hash(klo, khi)) && probe_from(a, klo, khi);
    } else if (P.state == 4) {
        present = sorted_contains(a, klo, khi);
    } else {
        const int v = bucket_verdict(a, P.w0, P.w1, klo, khi);
        present = v == 1 || (v == 2 && probe_from(a, klo, khi));
    }
    for (uint32_t att = 1; present; ++att) {
        if (att >= (uint32_t)kRejectCap) {
            atomicMin(a.err_slot, (unsigned long long)P.slot);
            break;
        }
        zero_candidate<D>(a, P.slot, att, o.c);
        o.attempts = (int)att + 1;
        first_bucket<D>(a, o.c, klo, khi);
        present = probe_from(a, klo, khi);
    }
    return o;
}

// Draw the sample of local slot `s` (0 <= s < p: nonzero slot s; p <= s < p+q:
// zero slot s-p).  Pure function of (seed, rank, kind, it, slot) and the tensor.
template <typename T, int D>
__device__ __forceinline__ Sample<T, D> draw_sample(const SampleArgs& a, int64_t s) {
    return resolve_sample<T, D>(a, issue_sample<T, D>(a, s));
}

}  // namespace gcp
