// ingest.cu -- row a0 (untimed setup): host COO -> device, validation, canonical
// lexicographic order (reading R15), duplicate check, AoS
// records, and the zero-test structure: an open-addressing hash set of block
// keys or the sorted key array (row f4).
//
// Memory-lean for billion-nonzero tensors: the host int64 coordinates stream
// through a fixed staging buffer and are converted on the fly to 32-bit local
// coordinates; the sort carries a 32-bit permutation when N < 2^32; the
// records and the hash set are built after the sort scratch is released.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>

#include "device.cuh"
#include "gcp_internal.h"

namespace gcp {

struct KeyArgs {
    int d;
    int64_t lo[kMaxModes], hi[kMaxModes];
    uint64_t bdim[kMaxModes];
};

enum : unsigned { BAD_RANGE = 1u, BAD_VALUE = 2u, BAD_DUP = 4u };

// Validate a chunk of host-order nonzeros, store 32-bit local coordinates and
// the value in T, and form the mixed-radix block key
// ((c_1 b_2 + c_2) b_3 + ...) b_d + c_d with c = i - lo.
template <typename T, typename PermT>
__global__ void k_convert(const KeyArgs ka, int64_t base, int64_t n, const int64_t* __restrict__ subs,
                          const double* __restrict__ vals, uint32_t* __restrict__ coords, T* __restrict__ valt,
                          uint64_t* __restrict__ klo, uint64_t* __restrict__ khi, PermT* __restrict__ perm,
                          unsigned* flags) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t gx = base + x;
        unsigned __int128 key = 0;
        unsigned bad = 0;
        for (int k = 0; k < ka.d; ++k) {
            const int64_t i = subs[x * ka.d + k];
            if (i < ka.lo[k] || i >= ka.hi[k]) {
                bad |= BAD_RANGE;
                coords[gx * ka.d + k] = 0;
                continue;
            }
            const uint64_t c = (uint64_t)(i - ka.lo[k]);
            coords[gx * ka.d + k] = (uint32_t)c;
            key = key * ka.bdim[k] + c;
        }
        const double v = vals[x];
        if (!isfinite(v)) bad |= BAD_VALUE;
        if (bad) atomicOr(flags, bad);
        valt[gx] = (T)v;
        klo[gx] = (uint64_t)key;
        if (khi) khi[gx] = (uint64_t)(key >> 64);
        perm[gx] = (PermT)gx;
    }
}

template <typename PermT>
__global__ void k_gather_u64(int64_t n, const PermT* __restrict__ perm, const uint64_t* __restrict__ in,
                             uint64_t* __restrict__ out) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x)
        out[x] = in[perm[x]];
}

// keys of the canonical order, recomputed from the local coordinates
template <typename PermT>
__global__ void k_sorted_keys(const KeyArgs ka, int64_t n, const PermT* __restrict__ perm,
                              const uint32_t* __restrict__ coords, uint64_t* __restrict__ klo,
                              uint64_t* __restrict__ khi) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t src = (int64_t)perm[x];
        unsigned __int128 key = 0;
        for (int k = 0; k < ka.d; ++k) key = key * ka.bdim[k] + coords[src * ka.d + k];
        klo[x] = (uint64_t)key;
        if (khi) khi[x] = (uint64_t)(key >> 64);
    }
}

__global__ void k_dupcheck(int64_t n, const uint64_t* __restrict__ klo, const uint64_t* __restrict__ khi,
                           unsigned* flags) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x + 1; x < n; x += (int64_t)gridDim.x * blockDim.x)
        if (klo[x] == klo[x - 1] && (!khi || khi[x] == khi[x - 1])) atomicOr(flags, BAD_DUP);
}

// Canonical AoS record n = [value][local coords][pad] of nonzero perm[n].
template <typename T, typename PermT>
__global__ void k_records(int d, int64_t n, int rec_words, const PermT* __restrict__ perm,
                          const uint32_t* __restrict__ coords, const T* __restrict__ valt, uint32_t* __restrict__ rec) {
    constexpr int VW = (int)(sizeof(T) / 4);
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t src = (int64_t)perm[x];
        uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const T v = valt[src];
        memcpy(w, &v, sizeof(T));
        for (int k = 0; k < d; ++k) w[VW + k] = coords[src * d + k];
        uint4* dst = reinterpret_cast<uint4*>(rec + x * rec_words);
        dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
        if (rec_words == 8) dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
    }
}

struct alignas(16) Key128 { uint64_t lo, hi; };

__global__ void k_hash_insert(int64_t n, const uint64_t* __restrict__ klo, const uint64_t* __restrict__ khi,
                              uint64_t* h, uint64_t mask) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
        if (!khi) {
            const uint64_t key = klo[x];
            uint64_t s = (hash_key(key, 0) & mask) & ~3ull;
            for (;;) {
                const unsigned long long prev =
                    atomicCAS(reinterpret_cast<unsigned long long*>(h + s), kEmpty, (unsigned long long)key);
                if (prev == kEmpty || prev == key) break;
                s = (s + 1) & mask;
            }
        } else {
            Key128 key{klo[x], khi[x]};
            uint64_t s = (hash_key(key.lo, key.hi) & mask) & ~1ull;
            const Key128 empty{kEmpty, kEmpty};
            for (;;) {
                Key128 prev = atomicCAS(reinterpret_cast<Key128*>(h + 2 * s), empty, key);
                if ((prev.lo == kEmpty && prev.hi == kEmpty) || (prev.lo == key.lo && prev.hi == key.hi)) break;
                s = (s + 1) & mask;
            }
        }
    }
}

// blocked Bloom filter (device.cuh filter_maybe): one bit in each u64 of the key's sector
__global__ void k_filter_insert(int64_t n, const uint64_t* __restrict__ klo, const uint64_t* __restrict__ khi,
                                unsigned long long* __restrict__ f, uint64_t mask) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t fh = filter_hash(klo[x], khi ? khi[x] : 0);
        unsigned long long* sec = f + 4 * (fh & mask);
#pragma unroll
        for (int i = 0; i < 4; ++i) atomicOr(sec + i, 1ull << ((fh >> (32 + 6 * i)) & 63));
    }
}

// Filter size: ~16 bits per key in a power-of-two number of 32-B sectors,
// capped at min(64 MB, 0.55 L2) so it stays L2-resident next to the factors;
// off below min_bits = 4 per key (c4 / c5 have no filter at all).  c2 gets 5.4
// bits per key (~8% "maybe"): K2 1.204 -> 1.177 ms against the plain hash
// probe under the final K2 geometry, and 1e7 fewer DRAM bucket reads per
// launch keep the clocks off the power cap (profiles/r02aa_*; round 1, with one
// round of row loads in flight, measured it the other way and kept it off).
// GCP_FILTER=0 disables it, GCP_FILTER_MB sets the cap, GCP_FILTER_MINBITS the
// threshold.
static uint64_t filter_sectors_for(const gcp_ctx* c, int64_t nnz, int min_bits) {
    const char* env = getenv("GCP_FILTER");
    if ((env && std::string(env) == "0") || nnz <= 0) return 0;
    const char* mb = getenv("GCP_FILTER_MB");
    const double cap_mb = mb ? atof(mb) : 64.0;
    const uint64_t cap = std::min<uint64_t>((uint64_t)(cap_mb * 1048576.0), (uint64_t)(c->l2_bytes * 0.55));
    const uint64_t want = (uint64_t)nnz * 2;
    uint64_t bytes = 32;
    while (bytes < want && bytes * 2 <= cap) bytes <<= 1;
    const char* mbits = getenv("GCP_FILTER_MINBITS");   // A/B switch for the bits-per-key threshold
    if (mbits) min_bits = atoi(mbits);
    if (bytes * 8 < (uint64_t)nnz * min_bits) return 0;
    return bytes / 32;
}

// sorted key array for the binary-search zero test (row f4): u64, or (lo, hi) pairs
__global__ void k_store_keys(int64_t n, const uint64_t* __restrict__ klo, const uint64_t* __restrict__ khi,
                             uint64_t* __restrict__ out) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
        if (khi) {
            out[2 * x] = klo[x];
            out[2 * x + 1] = khi[x];
        } else {
            out[x] = klo[x];
        }
    }
}

__global__ void k_contains(const KeyArgs ka, int64_t n, const int64_t* __restrict__ coords, const SampleArgs sa,
                           int8_t* out) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
        unsigned __int128 key = 0;
        for (int k = 0; k < ka.d; ++k) key = key * ka.bdim[k] + (uint64_t)(coords[x * ka.d + k] - ka.lo[k]);
        out[x] = probe_from(sa, (uint64_t)key, (uint64_t)(key >> 64));
    }
}

// ---- lean path (billion-nonzero blocks, u64 keys): sort (key, value) pairs
// directly -- no coordinate array, no permutation -- then decode the records
// from the sorted keys (the key is the mixed-radix block index, so the local
// coordinates are its digits).
template <typename T>
__global__ void k_convert_lean(const KeyArgs ka, int64_t base, int64_t n, const int64_t* __restrict__ subs,
                               const double* __restrict__ vals, T* __restrict__ valt, uint64_t* __restrict__ keys,
                               unsigned* flags) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
        uint64_t key = 0;
        unsigned bad = 0;
        for (int k = 0; k < ka.d; ++k) {
            const int64_t i = subs[x * ka.d + k];
            if (i < ka.lo[k] || i >= ka.hi[k]) {
                bad |= BAD_RANGE;
                continue;
            }
            key = key * ka.bdim[k] + (uint64_t)(i - ka.lo[k]);
        }
        const double v = vals[x];
        if (!isfinite(v)) bad |= BAD_VALUE;
        if (bad) atomicOr(flags, bad);
        valt[base + x] = (T)v;
        keys[base + x] = key;
    }
}

template <typename T>
__global__ void k_records_from_keys(const KeyArgs ka, int64_t n, int rec_words, const uint64_t* __restrict__ keys,
                                    const T* __restrict__ valt, uint32_t* __restrict__ rec) {
    constexpr int VW = (int)(sizeof(T) / 4);
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
        uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const T v = valt[x];
        memcpy(w, &v, sizeof(T));
        uint64_t key = keys[x];
        for (int k = ka.d - 1; k > 0; --k) {
            w[VW + k] = (uint32_t)(key % ka.bdim[k]);
            key /= ka.bdim[k];
        }
        w[VW] = (uint32_t)key;
        uint4* dst = reinterpret_cast<uint4*>(rec + x * rec_words);
        dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
        if (rec_words == 8) dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
    }
}

// hash set of u64 block keys recomputed from the records (the key array is
// already freed on the lean path)
__global__ void k_hash_insert_rec(const KeyArgs ka, int64_t n, int rec_words, int val_words,
                                  const uint32_t* __restrict__ rec, uint64_t* h, uint64_t mask) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t* r = rec + x * rec_words + val_words;
        uint64_t key = r[0];
        for (int k = 1; k < ka.d; ++k) key = key * ka.bdim[k] + r[k];
        uint64_t s = (hash_key(key, 0) & mask) & ~3ull;
        for (;;) {
            const unsigned long long prev =
                atomicCAS(reinterpret_cast<unsigned long long*>(h + s), kEmpty, (unsigned long long)key);
            if (prev == kEmpty || prev == key) break;
            s = (s + 1) & mask;
        }
    }
}

static KeyArgs key_args(const gcp_ctx* c) {
    KeyArgs ka;
    ka.d = c->d;
    for (int k = 0; k < kMaxModes; ++k) {
        ka.lo[k] = k < c->d ? c->lo[k] : 0;
        ka.hi[k] = k < c->d ? c->hi[k] : 0;
        ka.bdim[k] = k < c->d ? (uint64_t)(c->hi[k] - c->lo[k]) : 1;
    }
    return ka;
}

static int bits_for(unsigned __int128 v) {   // bits needed to represent v - 1 (v >= 1)
    int b = 0;
    unsigned __int128 x = v - 1;
    while (x) { ++b; x >>= 1; }
    return b;
}

cudaError_t launch_contains(gcp_ctx* c, int64_t n, const int64_t* coords, int8_t* out) {
    if (n == 0) return cudaSuccess;
    const KeyArgs ka = key_args(c);
    SampleArgs sa{};
    sa.N = c->N;
    sa.hash = c->d_hash;
    sa.hash_mask = c->hash_slots - 1;
    sa.key128 = c->key128;
    sa.member_sorted = c->member == GCP_MEMBER_SORTED;
    sa.keys = c->d_keys;
    k_contains<<<(int)std::min<int64_t>((n + 255) / 256, 65535), 256, 0, c->stream>>>(ka, n, coords, sa, out);
    return cudaGetLastError();
}


#define CK(x)                                              \
    do {                                                   \
        cudaError_t e_ = (x);                              \
        if (e_ != cudaSuccess) { err = e_; goto cleanup; } \
    } while (0)

// Ingest scratch (staging, keys, permutations, sort temp) comes from a pool of
// its own: repeated ingests of similar size find their blocks again instead of
// fragmenting the default pool that holds the tensor and the model (which made
// every few ingests map fresh memory).  Trimmed after an ingest when the
// device is short of free memory, and by gmalloc when an allocation fails.
static cudaError_t scratch_pool(gcp_ctx* c) {
    if (c->scratch_pool) return cudaSuccess;
    cudaMemPoolProps props;
    memset(&props, 0, sizeof(props));
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = c->dev;
    cudaError_t e = cudaMemPoolCreate(&c->scratch_pool, &props);
    if (e != cudaSuccess) return e;
    uint64_t thr = UINT64_MAX;
    return cudaMemPoolSetAttribute(c->scratch_pool, cudaMemPoolAttrReleaseThreshold, &thr);
}
template <typename P>
static cudaError_t smalloc(gcp_ctx* c, P** p, size_t bytes) {
    cudaError_t e = scratch_pool(c);
    if (e != cudaSuccess) return e;
    return cudaMallocFromPoolAsync(reinterpret_cast<void**>(p), bytes, c->scratch_pool, c->stream);
}
static void sfree(gcp_ctx* c, void* p) {
    if (p) cudaFreeAsync(p, c->stream);
}
static void scratch_trim_if_tight(gcp_ctx* c) {
    size_t fr = 0, tot = 0;
    if (!c->scratch_pool || cudaMemGetInfo(&fr, &tot) != cudaSuccess) return;
    // keep the scratch mapped for the next ingest unless the device is short of
    // memory (gmalloc also trims it and retries when a later allocation fails)
    if (fr < tot / 8) {
        cudaStreamSynchronize(c->stream);
        cudaMemPoolTrimTo(c->scratch_pool, 0);
    }
}

template <typename T, typename PermT>
static gcp_status ingest_impl(gcp_ctx* c, const gcp_ctx* g, int64_t nnz, const int64_t* subs_h,
                              const double* vals_h) {
    const KeyArgs ka = key_args(g);
    const int d = g->d;
    cudaStream_t st = c->stream;
    cudaError_t err = cudaSuccess;
    gcp_status status = GCP_OK;
    const int kbits = bits_for(g->M > 0 ? g->M : 1);
    const bool k128 = kbits > 64;
    const bool sorted_member = c->member == GCP_MEMBER_SORTED;
    const int rec_words = ((int)(sizeof(T) / 4) + d <= 4) ? 4 : 8;
    const int nb = (int)std::min<int64_t>(std::max<int64_t>((nnz + 255) / 256, 1), (int64_t)c->sm_count * 16);
    const int64_t chunk = std::min<int64_t>(std::max<int64_t>(nnz, 1), (int64_t)1 << 26);
    uint64_t slots = 4;
    if (!sorted_member) {
        const uint64_t need = (uint64_t)std::ceil((double)std::max<int64_t>(nnz, 1) / kHashLoad);
        while (slots < need) slots <<= 1;
    }
    const size_t kw = k128 ? 2 : 1;   // key words
    unsigned flags = 0;
    unsigned* d_flags = nullptr;
    int64_t* d_sc = nullptr;
    double* d_vc = nullptr;
    uint32_t* coords = nullptr;
    T* valt = nullptr;
    uint64_t *k0 = nullptr, *k1 = nullptr, *h0 = nullptr, *h1 = nullptr;
    PermT *p0 = nullptr, *p1 = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    PermT* perm = nullptr;
    uint64_t *skl = nullptr, *skh = nullptr;
    uint32_t* new_rec = nullptr;
    uint64_t* new_hash = nullptr;
    uint64_t* new_keys = nullptr;
    uint64_t* new_filter = nullptr;
    const uint64_t fsect = filter_sectors_for(c, nnz, 4);
    // diagnostics: GCP_INGEST_TRACE=1 syncs after each phase and prints its time
    const char* trace_env = getenv("GCP_INGEST_TRACE");
    const bool trace = trace_env && trace_env[0] == '1';
    auto t_last = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (!trace) return;
        cudaStreamSynchronize(st);
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[gcp ingest] %-28s %9.1f ms\n", what,
                std::chrono::duration<double, std::milli>(now - t_last).count());
        t_last = now;
    };

    CK(smalloc(c, &d_flags, sizeof(unsigned)));
    CK(cudaMemsetAsync(d_flags, 0, sizeof(unsigned), st));
    if (nnz > 0) {
        // 1) stream the host COO through the staging buffer, converting on the fly
        CK(smalloc(c, &coords, (size_t)nnz * d * 4));
        CK(smalloc(c, &valt, (size_t)nnz * sizeof(T)));
        CK(smalloc(c, &k0, (size_t)nnz * 8));
        if (k128) CK(smalloc(c, &h0, (size_t)nnz * 8));
        CK(smalloc(c, &p0, (size_t)nnz * sizeof(PermT)));
        CK(smalloc(c, &d_sc, (size_t)chunk * d * 8));
        CK(smalloc(c, &d_vc, (size_t)chunk * 8));
        for (int64_t b = 0; b < nnz; b += chunk) {
            const int64_t n = std::min(chunk, nnz - b);
            CK(cudaMemcpyAsync(d_sc, subs_h + b * d, (size_t)n * d * 8, cudaMemcpyDefault, st));
            CK(cudaMemcpyAsync(d_vc, vals_h + b, (size_t)n * 8, cudaMemcpyDefault, st));
            k_convert<T, PermT><<<nb, 256, 0, st>>>(ka, b, n, d_sc, d_vc, coords, valt, k0, h0, p0, d_flags);
            CK(cudaGetLastError());
            c->launches++;
        }
        CK(cudaMemcpyAsync(&flags, d_flags, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        mark("H2D + convert");
        sfree(c, d_sc); d_sc = nullptr;
        sfree(c, d_vc); d_vc = nullptr;
        if (flags & BAD_RANGE) { status = set_error(GCP_E_RANGE, "gcp_tensor_create: coordinate outside dims / block"); goto cleanup; }
        if (flags & BAD_VALUE) { status = set_error(GCP_E_ARG, "gcp_tensor_create: non-finite value"); goto cleanup; }
        // 2) LSD radix sort of (key, perm): low word, then stably the high word
        CK(smalloc(c, &k1, (size_t)nnz * 8));
        CK(smalloc(c, &p1, (size_t)nnz * sizeof(PermT)));
        {
            cub::DoubleBuffer<uint64_t> keys(k0, k1);
            cub::DoubleBuffer<PermT> pm(p0, p1);
            const int lo_bits = k128 ? 64 : std::max(kbits, 1);
            CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, pm, nnz, 0, lo_bits, st));
            CK(smalloc(c, &tmp, tmp_bytes));
            CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, pm, nnz, 0, lo_bits, st));
            if (k128) {
                // high words in the current order, then a stable sort on them
                uint64_t* hbuf = keys.Alternate();
                k_gather_u64<PermT><<<nb, 256, 0, st>>>(nnz, pm.Current(), h0, hbuf);
                CK(cudaGetLastError());
                c->launches++;
                cub::DoubleBuffer<uint64_t> hk(hbuf, keys.Current());
                size_t tb2 = 0;
                CK(cub::DeviceRadixSort::SortPairs(nullptr, tb2, hk, pm, nnz, 0, kbits - 64, st));
                if (tb2 > tmp_bytes) {
                    sfree(c, tmp);
                    tmp = nullptr;
                    CK(smalloc(c, &tmp, tb2));
                    tmp_bytes = tb2;
                }
                CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, hk, pm, nnz, 0, kbits - 64, st));
            }
            perm = pm.Current();
            // keys in canonical order, recomputed from the coordinates into the
            // (now free) key buffers
            skl = k0;
            skh = k128 ? h0 : nullptr;
            k_sorted_keys<PermT><<<nb, 256, 0, st>>>(ka, nnz, perm, coords, skl, skh);
            CK(cudaGetLastError());
            c->launches++;
        }
        mark("radix sort + sorted keys");
        sfree(c, tmp); tmp = nullptr;
        sfree(c, k1); k1 = nullptr;
        sfree(c, perm == p0 ? p1 : p0);
        if (perm == p0) p1 = nullptr; else p0 = nullptr;
        // 3) duplicates, records
        k_dupcheck<<<nb, 256, 0, st>>>(nnz, skl, skh, d_flags);
        CK(cudaGetLastError());
        c->launches++;
        CK(gmalloc(c, &new_rec, (size_t)nnz * rec_words * 4));
        k_records<T, PermT><<<nb, 256, 0, st>>>(d, nnz, rec_words, perm, coords, valt, new_rec);
        CK(cudaGetLastError());
        c->launches++;
        CK(cudaMemcpyAsync(&flags, d_flags, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (flags & BAD_DUP) { status = set_error(GCP_E_DUP, "gcp_tensor_create: duplicate coordinates"); goto cleanup; }
        sfree(c, coords); coords = nullptr;
        sfree(c, valt); valt = nullptr;
        sfree(c, p0); p0 = nullptr;
        sfree(c, p1); p1 = nullptr;
    } else {
        CK(gmalloc(c, &new_rec, (size_t)rec_words * 4));
    }
    mark("dup check + records");
    // 4) zero-test structure
    CK(gmalloc(c, &new_hash, (size_t)slots * 8 * kw));
    CK(cudaMemsetAsync(new_hash, 0xFF, (size_t)slots * 8 * kw, st));
    CK(gmalloc(c, &new_keys, (size_t)(sorted_member ? std::max<int64_t>(nnz, 1) : 1) * 8 * kw));
    if (nnz > 0) {
        if (sorted_member) k_store_keys<<<nb, 256, 0, st>>>(nnz, skl, skh, new_keys);
        else k_hash_insert<<<nb, 256, 0, st>>>(nnz, skl, skh, new_hash, slots - 1);
        CK(cudaGetLastError());
        c->launches++;
        if (fsect) {
            CK(gmalloc(c, &new_filter, (size_t)fsect * 32));
            CK(cudaMemsetAsync(new_filter, 0, (size_t)fsect * 32, st));
            k_filter_insert<<<nb, 256, 0, st>>>(nnz, skl, skh, (unsigned long long*)new_filter, fsect - 1);
            CK(cudaGetLastError());
            c->launches++;
        }
    }
    CK(cudaStreamSynchronize(st));
    mark("hash / keys / filter");

cleanup:
    sfree(c, d_flags); sfree(c, d_sc); sfree(c, d_vc); sfree(c, coords); sfree(c, valt);
    sfree(c, k0); sfree(c, k1); sfree(c, h0); sfree(c, h1); sfree(c, p0); sfree(c, p1); sfree(c, tmp);
    if (err != cudaSuccess || status != GCP_OK) {
        gfree(c, new_rec);
        gfree(c, new_hash);
        gfree(c, new_keys);
        gfree(c, new_filter);
        if (err == cudaErrorMemoryAllocation) {
            cudaGetLastError();
            return set_error(GCP_E_OOM, "gcp_tensor_create: out of device memory");
        }
        if (err != cudaSuccess) return cuda_fail(c, err, "gcp_tensor_create");
        return status;
    }
    // commit
    gfree(c, c->d_rec);
    gfree(c, c->d_hash);
    gfree(c, c->d_keys);
    gfree(c, c->d_filter);
    c->d_filter = new_filter;
    c->filter_sectors = new_filter ? fsect : 0;
    c->d_rec = new_rec;
    c->d_hash = new_hash;
    c->d_keys = new_keys;
    c->key128 = k128 ? 1 : 0;
    c->val_words = (int)(sizeof(T) / 4);
    c->rec_words = rec_words;
    c->hash_slots = slots;
    c->lean_ingest = false;
    return GCP_OK;
}

// Lean ingest (row a0 for billion-nonzero blocks, e.g. c5's 4.69e9 nonzeros at
// one GPU): peak = 2 x (8 + sizeof(T)) B per nonzero during the sort, then
// records (16 B) + sorted keys + values; the hash set is built from the
// records after the keys and values are freed.  Same records, same keys, same
// membership answers as the standard path.
template <typename T>
static gcp_status ingest_lean(gcp_ctx* c, const gcp_ctx* g, int64_t nnz, const int64_t* subs_h,
                              const double* vals_h) {
    const KeyArgs ka = key_args(g);
    const int d = g->d;
    cudaStream_t st = c->stream;
    cudaError_t err = cudaSuccess;
    gcp_status status = GCP_OK;
    const int kbits = std::max(bits_for(g->M > 0 ? g->M : 1), 1);
    const bool sorted_member = c->member == GCP_MEMBER_SORTED;
    const int rec_words = ((int)(sizeof(T) / 4) + d <= 4) ? 4 : 8;
    const int nb = (int)std::min<int64_t>(std::max<int64_t>((nnz + 255) / 256, 1), (int64_t)c->sm_count * 16);
    const int64_t chunk = std::min<int64_t>(nnz, (int64_t)1 << 26);
    unsigned flags = 0;
    unsigned* d_flags = nullptr;
    int64_t* d_sc = nullptr;
    double* d_vc = nullptr;
    uint64_t *k0 = nullptr, *k1 = nullptr;
    T *v0 = nullptr, *v1 = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    uint64_t* skeys = nullptr;   // sorted keys (k0 or k1)
    T* svals = nullptr;
    uint32_t* new_rec = nullptr;
    uint64_t* new_hash = nullptr;
    uint64_t* new_keys = nullptr;
    uint64_t* new_filter = nullptr;
    uint64_t slots = 4;
    const uint64_t fsect = filter_sectors_for(c, nnz, 4);

    CK(smalloc(c, &d_flags, sizeof(unsigned)));
    CK(cudaMemsetAsync(d_flags, 0, sizeof(unsigned), st));
    // 1) stream the host COO through the staging buffer: keys + values
    CK(gmalloc(c, &k0, (size_t)nnz * 8));
    CK(smalloc(c, &v0, (size_t)nnz * sizeof(T)));
    CK(smalloc(c, &d_sc, (size_t)chunk * d * 8));
    CK(smalloc(c, &d_vc, (size_t)chunk * 8));
    for (int64_t b = 0; b < nnz; b += chunk) {
        const int64_t n = std::min(chunk, nnz - b);
        CK(cudaMemcpyAsync(d_sc, subs_h + b * d, (size_t)n * d * 8, cudaMemcpyDefault, st));
        CK(cudaMemcpyAsync(d_vc, vals_h + b, (size_t)n * 8, cudaMemcpyDefault, st));
        k_convert_lean<T><<<nb, 256, 0, st>>>(ka, b, n, d_sc, d_vc, v0, k0, d_flags);
        CK(cudaGetLastError());
        c->launches++;
    }
    CK(cudaMemcpyAsync(&flags, d_flags, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    sfree(c, d_sc); d_sc = nullptr;
    sfree(c, d_vc); d_vc = nullptr;
    if (flags & BAD_RANGE) { status = set_error(GCP_E_RANGE, "gcp_tensor_create: coordinate outside dims / block"); goto cleanup; }
    if (flags & BAD_VALUE) { status = set_error(GCP_E_ARG, "gcp_tensor_create: non-finite value"); goto cleanup; }
    // 2) radix sort of (key, value) pairs over the key's bits (64-bit item count)
    CK(gmalloc(c, &k1, (size_t)nnz * 8));
    CK(smalloc(c, &v1, (size_t)nnz * sizeof(T)));
    {
        cub::DoubleBuffer<uint64_t> keys(k0, k1);
        cub::DoubleBuffer<T> vs(v0, v1);
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, vs, nnz, 0, kbits, st));
        CK(smalloc(c, &tmp, tmp_bytes));
        CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, vs, nnz, 0, kbits, st));
        skeys = keys.Current();
        svals = vs.Current();
    }
    sfree(c, tmp); tmp = nullptr;
    if (skeys == k0) { gfree(c, k1); k1 = nullptr; } else { gfree(c, k0); k0 = nullptr; }
    if (svals == v0) { sfree(c, v1); v1 = nullptr; } else { sfree(c, v0); v0 = nullptr; }
    // 3) duplicates, records decoded from the keys
    k_dupcheck<<<nb, 256, 0, st>>>(nnz, skeys, nullptr, d_flags);
    CK(cudaGetLastError());
    c->launches++;
    CK(gmalloc(c, &new_rec, (size_t)nnz * rec_words * 4));
    k_records_from_keys<T><<<nb, 256, 0, st>>>(ka, nnz, rec_words, skeys, svals, new_rec);
    CK(cudaGetLastError());
    c->launches++;
    CK(cudaMemcpyAsync(&flags, d_flags, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (flags & BAD_DUP) { status = set_error(GCP_E_DUP, "gcp_tensor_create: duplicate coordinates"); goto cleanup; }
    sfree(c, svals);
    v0 = v1 = nullptr;
    // 4) zero-test structure: the sorted keys themselves (row f4), or a hash set
    //    built from the records once the keys are gone
    if (fsect) {
        CK(gmalloc(c, &new_filter, (size_t)fsect * 32));
        CK(cudaMemsetAsync(new_filter, 0, (size_t)fsect * 32, st));
        k_filter_insert<<<nb, 256, 0, st>>>(nnz, skeys, nullptr, (unsigned long long*)new_filter, fsect - 1);
        CK(cudaGetLastError());
        c->launches++;
    }
    if (sorted_member) {
        new_keys = skeys;
        k0 = k1 = nullptr;
        CK(gmalloc(c, &new_hash, 32));
        CK(cudaMemsetAsync(new_hash, 0xFF, 32, st));
    } else {
        gfree(c, skeys);
        k0 = k1 = nullptr;
        CK(cudaStreamSynchronize(st));
        cudaMemPoolTrimTo(c->scratch_pool, 0);
        {
            const uint64_t need = (uint64_t)std::ceil((double)nnz / kHashLoad);
            while (slots < need) slots <<= 1;
            // memory-tight blocks take a fuller table (load <= 0.75): keep 10% of
            // the device (>= 16 GB) free for the model
            size_t fr = 0, tot = 0;
            cudaMemGetInfo(&fr, &tot);
            const double reserve = std::max(16.0 * (1 << 30), 0.1 * (double)tot);
            while ((double)slots * 8 > (double)fr - reserve && (double)nnz / (double)(slots / 2) <= 0.75)
                slots >>= 1;
        }
        CK(gmalloc(c, &new_hash, (size_t)slots * 8));
        CK(cudaMemsetAsync(new_hash, 0xFF, (size_t)slots * 8, st));
        k_hash_insert_rec<<<nb, 256, 0, st>>>(ka, nnz, rec_words, (int)(sizeof(T) / 4), new_rec, new_hash, slots - 1);
        CK(cudaGetLastError());
        c->launches++;
        CK(gmalloc(c, &new_keys, 8));
    }
    CK(cudaStreamSynchronize(st));

cleanup:
    sfree(c, d_flags); sfree(c, d_sc); sfree(c, d_vc); sfree(c, tmp);
    sfree(c, v0); sfree(c, v1);
    gfree(c, k0); gfree(c, k1);
    if (err != cudaSuccess || status != GCP_OK) {
        gfree(c, new_rec);
        gfree(c, new_hash);
        gfree(c, new_keys);
        gfree(c, new_filter);
        if (err == cudaErrorMemoryAllocation) {
            cudaGetLastError();
            return set_error(GCP_E_OOM, "gcp_tensor_create: out of device memory (lean ingest)");
        }
        if (err != cudaSuccess) return cuda_fail(c, err, "gcp_tensor_create");
        return status;
    }
    gfree(c, c->d_rec);
    gfree(c, c->d_hash);
    gfree(c, c->d_keys);
    gfree(c, c->d_filter);
    c->d_filter = new_filter;
    c->filter_sectors = new_filter ? fsect : 0;
    c->d_rec = new_rec;
    c->d_hash = new_hash;
    c->d_keys = new_keys;
    c->key128 = 0;
    c->val_words = (int)(sizeof(T) / 4);
    c->rec_words = rec_words;
    c->hash_slots = sorted_member ? 4 : slots;
    c->lean_ingest = true;
    return GCP_OK;
}

gcp_status ingest(gcp_ctx* c, const gcp_ctx* g, int64_t nnz, const int64_t* subs_h, const double* vals_h) {
    const bool p32 = nnz < ((int64_t)1 << 32);
    gcp_status st;
    // the lean path (u64 keys only): when the standard path's scratch (coords,
    // values, keys and permutations, double-buffered) would not fit, or forced
    // by GCP_INGEST=lean (tests); GCP_INGEST=standard forces the other
    const char* env = getenv("GCP_INGEST");
    const std::string mode = env ? env : "auto";
    const bool k64 = bits_for(g->M > 0 ? g->M : 1) <= 64;
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    const double std_bytes = (double)nnz * (g->d * 4 + c->tsize + 16 + 2 * (p32 ? 4 : 8) + c->tsize * 4);
    const bool lean = k64 && nnz > 0 && (mode == "lean" || (mode != "standard" && std_bytes > 0.8 * (double)fr));
    if (lean) {
        st = c->prec == GCP_FP32 ? ingest_lean<float>(c, g, nnz, subs_h, vals_h)
                                 : ingest_lean<double>(c, g, nnz, subs_h, vals_h);
        scratch_trim_if_tight(c);
        return st;
    }
    if (c->prec == GCP_FP32)
        st = p32 ? ingest_impl<float, uint32_t>(c, g, nnz, subs_h, vals_h)
                 : ingest_impl<float, uint64_t>(c, g, nnz, subs_h, vals_h);
    else
        st = p32 ? ingest_impl<double, uint32_t>(c, g, nnz, subs_h, vals_h)
                 : ingest_impl<double, uint64_t>(c, g, nnz, subs_h, vals_h);
    scratch_trim_if_tight(c);
    return st;
}

}  // namespace gcp
