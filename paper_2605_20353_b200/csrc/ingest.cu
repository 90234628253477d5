// ingest.cu -- row a0 (untimed setup): host COO -> device, validation, canonical
// lexicographic order (reading R15), duplicate check, AoS
// records, and the open-addressing hash set of block keys.
#include <cub/device/device_radix_sort.cuh>

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

// Validate every coordinate / value and form the mixed-radix block key
// ((c_1 b_2 + c_2) b_3 + ...) b_d + c_d of the local coordinates c = i - lo.
__global__ void k_keys(const KeyArgs ka, int64_t n, const int64_t* __restrict__ subs,
                       const double* __restrict__ vals, uint64_t* __restrict__ klo, uint64_t* __restrict__ khi,
                       uint64_t* __restrict__ perm, unsigned* flags) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
        unsigned __int128 key = 0;
        unsigned bad = 0;
        for (int k = 0; k < ka.d; ++k) {
            const int64_t i = subs[x * ka.d + k];
            if (i < ka.lo[k] || i >= ka.hi[k]) { bad |= BAD_RANGE; break; }
            key = key * ka.bdim[k] + (uint64_t)(i - ka.lo[k]);
        }
        if (!isfinite(vals[x])) bad |= BAD_VALUE;
        if (bad) atomicOr(flags, bad);
        klo[x] = (uint64_t)key;
        if (khi) khi[x] = (uint64_t)(key >> 64);
        perm[x] = (uint64_t)x;
    }
}

__global__ void k_gather_hi(int64_t n, const uint64_t* __restrict__ perm, const uint64_t* __restrict__ hi_in,
                            uint64_t* __restrict__ hi_out) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x)
        hi_out[x] = hi_in[perm[x]];
}

__global__ void k_gather_lo(int64_t n, const uint64_t* __restrict__ perm, const uint64_t* __restrict__ lo_in,
                            uint64_t* __restrict__ lo_out) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x)
        lo_out[x] = lo_in[perm[x]];
}

__global__ void k_dupcheck(int64_t n, const uint64_t* __restrict__ klo, const uint64_t* __restrict__ khi,
                           unsigned* flags) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x + 1; x < n; x += (int64_t)gridDim.x * blockDim.x)
        if (klo[x] == klo[x - 1] && (!khi || khi[x] == khi[x - 1])) atomicOr(flags, BAD_DUP);
}

// Canonical AoS record n = [value][local coords][pad] of nonzero perm[n].
template <typename T>
__global__ void k_records(int d, int64_t n, int rec_words, int val_words, const KeyArgs ka,
                          const uint64_t* __restrict__ perm, const int64_t* __restrict__ subs,
                          const double* __restrict__ vals, uint32_t* __restrict__ rec) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t src = (int64_t)perm[x];
        uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const T v = (T)vals[src];
        memcpy(w, &v, sizeof(T));
        for (int k = 0; k < d; ++k) w[val_words + k] = (uint32_t)(subs[src * d + k] - ka.lo[k]);
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

gcp_status ingest(gcp_ctx* c, const gcp_ctx* g, int64_t nnz, const int64_t* subs_h, const double* vals_h) {
    // g: staged geometry (d, lo, hi, M) of the new tensor; c: the context (stream, scratch)
    const KeyArgs ka = key_args(g);
    const int d = g->d;
    cudaStream_t st = c->stream;
    cudaError_t err = cudaSuccess;
    gcp_status status = GCP_OK;
    int64_t* d_subs = nullptr;
    double* d_vals = nullptr;
    uint64_t *k0 = nullptr, *k1 = nullptr, *p0 = nullptr, *p1 = nullptr, *hi0 = nullptr, *hi1 = nullptr;
    unsigned* d_flags = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    unsigned flags = 0;
    const int nb = (int)std::min<int64_t>(std::max<int64_t>((nnz + 255) / 256, 1), (int64_t)c->sm_count * 16);
    const int kbits = bits_for(g->M > 0 ? g->M : 1);
    const bool k128 = kbits > 64;
    const uint64_t slots_needed = (uint64_t)std::ceil((double)(nnz > 0 ? nnz : 1) / kHashLoad);
    uint64_t slots = 4;
    while (slots < slots_needed) slots <<= 1;
    const int tw = (c->prec == GCP_FP32) ? 4 : 8;

    uint32_t* new_rec = nullptr;
    uint64_t* new_hash = nullptr;
    uint64_t* new_keys = nullptr;
    const bool sorted_member = c->member == GCP_MEMBER_SORTED;
    const int val_words = tw / 4;
    const int rec_words = (val_words + d <= 4) ? 4 : 8;
    if (sorted_member) slots = 4;   // no hash set: a 4-slot empty table keeps the pointer valid

    CK(cudaMalloc(&d_flags, sizeof(unsigned)));
    CK(cudaMemsetAsync(d_flags, 0, sizeof(unsigned), st));
    CK(cudaMalloc(&new_rec, (size_t)std::max<int64_t>(nnz, 1) * rec_words * 4));
    CK(cudaMalloc(&new_hash, (size_t)slots * 8 * (k128 ? 2 : 1)));
    CK(cudaMemsetAsync(new_hash, 0xFF, (size_t)slots * 8 * (k128 ? 2 : 1), st));
    CK(cudaMalloc(&new_keys, (size_t)(sorted_member ? std::max<int64_t>(nnz, 1) : 1) * 8 * (k128 ? 2 : 1)));
    if (nnz > 0) {
        CK(cudaMalloc(&d_subs, (size_t)nnz * d * sizeof(int64_t)));
        CK(cudaMalloc(&d_vals, (size_t)nnz * sizeof(double)));
        CK(cudaMemcpyAsync(d_subs, subs_h, (size_t)nnz * d * sizeof(int64_t), cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(d_vals, vals_h, (size_t)nnz * sizeof(double), cudaMemcpyHostToDevice, st));
        CK(cudaMalloc(&k0, (size_t)nnz * 8));
        CK(cudaMalloc(&k1, (size_t)nnz * 8));
        CK(cudaMalloc(&p0, (size_t)nnz * 8));
        CK(cudaMalloc(&p1, (size_t)nnz * 8));
        if (k128) {
            CK(cudaMalloc(&hi0, (size_t)nnz * 8));
            CK(cudaMalloc(&hi1, (size_t)nnz * 8));
        }
        k_keys<<<nb, 256, 0, st>>>(ka, nnz, d_subs, d_vals, k0, hi0, p0, d_flags);
        CK(cudaGetLastError());
        c->launches++;
        CK(cudaMemcpyAsync(&flags, d_flags, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (flags & BAD_RANGE) { status = set_error(GCP_E_RANGE, "gcp_tensor_create: coordinate outside dims / block"); goto cleanup; }
        if (flags & BAD_VALUE) { status = set_error(GCP_E_ARG, "gcp_tensor_create: non-finite value"); goto cleanup; }
        {
            // LSD radix sort: (low 64 bits, perm), then stably by the high word
            cub::DoubleBuffer<uint64_t> keys(k0, k1), perm(p0, p1);
            const int lo_bits = k128 ? 64 : (kbits > 0 ? kbits : 1);
            CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, perm, nnz, 0, lo_bits, st));
            CK(cudaMalloc(&tmp, tmp_bytes));
            CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, perm, nnz, 0, lo_bits, st));
            uint64_t* sorted_lo = keys.Current();
            uint64_t* sorted_perm = perm.Current();
            uint64_t* sorted_hi = nullptr;
            if (k128) {
                // hi' = hi[perm]; sort (hi', perm) stably; then lo = key_lo[perm]
                uint64_t* other_perm = perm.Alternate();
                k_gather_hi<<<nb, 256, 0, st>>>(nnz, sorted_perm, hi0, hi1);
                CK(cudaGetLastError());
                c->launches++;
                cub::DoubleBuffer<uint64_t> hk(hi1, hi0), pp(sorted_perm, other_perm);
                size_t tb2 = 0;
                CK(cub::DeviceRadixSort::SortPairs(nullptr, tb2, hk, pp, nnz, 0, kbits - 64, st));
                if (tb2 > tmp_bytes) {
                    cudaFree(tmp);
                    tmp = nullptr;
                    CK(cudaMalloc(&tmp, tb2));
                    tmp_bytes = tb2;
                }
                CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, hk, pp, nnz, 0, kbits - 64, st));
                sorted_hi = hk.Current();
                sorted_perm = pp.Current();
                // recompute low words in the final order from the original keys
                uint64_t* lo_orig = (sorted_lo == k0) ? k1 : k0;   // scratch
                k_keys<<<nb, 256, 0, st>>>(ka, nnz, d_subs, d_vals, lo_orig, hk.Alternate(), pp.Alternate(),
                                           d_flags);
                CK(cudaGetLastError());
                c->launches++;
                k_gather_lo<<<nb, 256, 0, st>>>(nnz, sorted_perm, lo_orig, sorted_lo);
                CK(cudaGetLastError());
                c->launches++;
            }
            k_dupcheck<<<nb, 256, 0, st>>>(nnz, sorted_lo, sorted_hi, d_flags);
            CK(cudaGetLastError());
            c->launches++;
            if (c->prec == GCP_FP32)
                k_records<float><<<nb, 256, 0, st>>>(d, nnz, rec_words, val_words, ka, sorted_perm, d_subs,
                                                     d_vals, new_rec);
            else
                k_records<double><<<nb, 256, 0, st>>>(d, nnz, rec_words, val_words, ka, sorted_perm, d_subs,
                                                      d_vals, new_rec);
            CK(cudaGetLastError());
            c->launches++;
            if (sorted_member)
                k_store_keys<<<nb, 256, 0, st>>>(nnz, sorted_lo, sorted_hi, new_keys);
            else
                k_hash_insert<<<nb, 256, 0, st>>>(nnz, sorted_lo, sorted_hi, new_hash, slots - 1);
            CK(cudaGetLastError());
            c->launches++;
            CK(cudaMemcpyAsync(&flags, d_flags, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            if (flags & BAD_DUP) { status = set_error(GCP_E_DUP, "gcp_tensor_create: duplicate coordinates"); goto cleanup; }
        }
    }
    CK(cudaStreamSynchronize(st));

cleanup:
    cudaFree(d_subs); cudaFree(d_vals); cudaFree(k0); cudaFree(k1); cudaFree(p0); cudaFree(p1);
    cudaFree(hi0); cudaFree(hi1); cudaFree(tmp); cudaFree(d_flags);
    if (err != cudaSuccess || status != GCP_OK) {
        cudaFree(new_rec);
        cudaFree(new_hash);
        cudaFree(new_keys);
        if (err == cudaErrorMemoryAllocation) {
            cudaGetLastError();
            return set_error(GCP_E_OOM, "gcp_tensor_create: out of device memory");
        }
        if (err != cudaSuccess) return cuda_fail(c, err, "gcp_tensor_create");
        return status;
    }
    // commit
    cudaFree(c->d_rec);
    cudaFree(c->d_hash);
    cudaFree(c->d_keys);
    c->d_rec = new_rec;
    c->d_hash = new_hash;
    c->d_keys = new_keys;
    c->key128 = k128 ? 1 : 0;
    c->val_words = val_words;
    c->rec_words = rec_words;
    c->hash_slots = slots;
    return GCP_OK;
}

}  // namespace gcp
