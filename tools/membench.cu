// membench.cu -- random-access ceilings of the B200 memory system for the access
// patterns of the GCP hot path (development tool; not part of libgcp.so).
//
//   rand16_hbm : random 16-B loads from a 2 GiB array (COO record fetch pattern)
//   rand32_hbm : random 32-B loads (two 16-B halves of one sector; hash bucket)
//   rand64_l2  : random 64-B rows (4 lanes x 16 B) from a 2 MiB array (L2-resident factors)
//   red64_l2   : random 64-B vector red.add rows into a 2 MiB array (gradient scatter)
//   copy_hbm   : streaming float4 copy (reference)
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/membench tools/membench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

template <int ILP>
__global__ void rand_load(const uint4* __restrict__ a, uint64_t n, int64_t total, int words, uint32_t* sink) {
    uint32_t acc = 0;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = tid; i < total; i += nt * ILP) {
        uint4 v[ILP], u[ILP];
#pragma unroll
        for (int k = 0; k < ILP; ++k) {
            const uint64_t j = __umul64hi(mix(i + k * nt), n);
            v[k] = __ldg(a + j * words);
            if (words == 2) u[k] = __ldg(a + j * words + 1);
        }
#pragma unroll
        for (int k = 0; k < ILP; ++k) {
            acc += v[k].x ^ v[k].w;
            if (words == 2) acc += u[k].y;
        }
    }
    if (acc == 0x12345678u) *sink = acc;
}

// groups of 4 lanes read one 64-B row each
template <int ILP>
__global__ void rand_rows(const float4* __restrict__ a, uint64_t rows, int64_t total, float* sink) {
    float acc = 0.f;
    const int lane = threadIdx.x & 3;
    const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 2;
    const int64_t ng = ((int64_t)gridDim.x * blockDim.x) >> 2;
    for (int64_t i = g; i < total; i += ng * ILP) {
        float4 v[ILP];
#pragma unroll
        for (int k = 0; k < ILP; ++k) {
            const uint64_t r = __umul64hi(mix(i + k * ng), rows);
            v[k] = __ldg(a + r * 4 + lane);
        }
#pragma unroll
        for (int k = 0; k < ILP; ++k) acc += v[k].x + v[k].w;
    }
    if (acc == 1.2345f) *sink = acc;
}

__global__ void rand_red(float4* a, uint64_t rows, int64_t total) {
    const int lane = threadIdx.x & 3;
    const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 2;
    const int64_t ng = ((int64_t)gridDim.x * blockDim.x) >> 2;
    for (int64_t i = g; i < total; i += ng) {
        const uint64_t r = __umul64hi(mix(i), rows);
        float* p = reinterpret_cast<float*>(a + r * 4 + lane);
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f)
                     : "memory");
    }
}

// shared-memory privatisation candidate: random 64-B rows, 4 lanes x 4 scalar
// atomicAdd(float) each, into a per-CTA array of srows rows (dynamic smem)
__global__ void smem_red(float* out, int srows, int64_t total) {
    extern __shared__ float sh[];
    for (int i = threadIdx.x; i < srows * 16; i += blockDim.x) sh[i] = 0.f;
    __syncthreads();
    const int lane = threadIdx.x & 3;
    const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 2;
    const int64_t ng = ((int64_t)gridDim.x * blockDim.x) >> 2;
    for (int64_t i = g; i < total; i += ng) {
        const uint32_t r = __umulhi((uint32_t)mix(i), (uint32_t)srows);
        float* p = sh + r * 16 + lane * 4;
        atomicAdd(p, 1.f);
        atomicAdd(p + 1, 1.f);
        atomicAdd(p + 2, 1.f);
        atomicAdd(p + 3, 1.f);
    }
    __syncthreads();
    if (threadIdx.x == 0 && sh[0] == 1.2345f) out[0] = sh[1];
}

// K2's memory skeleton per sample (no Philox, no hash logic): optionally one
// random 16-B DRAM load (record / bucket), then 3 random 64-B row loads and 3
// random 64-B red.add.v4 rows in an L2-resident factor / gradient array, 4
// lanes per sample -- the combined L2 ceiling the fused kernel shares.
__global__ void k2_skeleton(const uint4* __restrict__ big, uint64_t nbig, const float4* __restrict__ A, float4* G,
                            uint64_t rows, int64_t total, int with_dram, float* sink) {
    const int lane = threadIdx.x & 3;
    const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 2;
    const int64_t ng = ((int64_t)gridDim.x * blockDim.x) >> 2;
    float acc = 0.f;
    for (int64_t i = g; i < total; i += ng) {
        uint64_t h = mix(i);
        uint32_t extra = 0;
        if (with_dram) {
            const uint4 v = __ldg(big + __umul64hi(h, nbig));
            extra = v.x & 1;
        }
        uint64_t r[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            h = mix(h + k + 1 + extra);
            r[k] = __umul64hi(h, rows / 3) + k * (rows / 3);
        }
        float4 a[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) a[k] = __ldg(A + r[k] * 4 + lane);
        const float m = a[0].x * a[1].x * a[2].x + a[0].y * a[1].y * a[2].y;
        acc += m;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            float* p = reinterpret_cast<float*>(G + r[k] * 4 + lane);
            const float4 o = a[(k + 1) % 3], q = a[(k + 2) % 3];
            asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(m * o.x * q.x),
                         "f"(m * o.y * q.y), "f"(m * o.z * q.z), "f"(m * o.w * q.w)
                         : "memory");
        }
    }
    if (acc == 1.2345f) *sink = acc;
}

// c4-shaped skeleton: factor rows DRAM-resident, A and G rows interleaved in
// one 128-B line (row r: A at float4 8r..8r+3, G at 8r+4..8r+7), 3 modes.
__global__ void k2_skeleton_dram(const uint4* __restrict__ big, uint64_t nbig, float4* AG, uint64_t rows,
                                 int64_t total, float* sink) {
    const int lane = threadIdx.x & 3;
    const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 2;
    const int64_t ng = ((int64_t)gridDim.x * blockDim.x) >> 2;
    float acc = 0.f;
    for (int64_t i = g; i < total; i += ng) {
        uint64_t h = mix(i);
        const uint4 v = __ldg(big + __umul64hi(h, nbig));
        uint64_t r[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            h = mix(h + k + 1 + (v.x & 1));
            r[k] = __umul64hi(h, rows / 3) + k * (rows / 3);
        }
        float4 a[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) a[k] = __ldg(AG + r[k] * 8 + lane);
        const float m = a[0].x * a[1].x * a[2].x + a[0].y * a[1].y * a[2].y;
        acc += m;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            float* p = reinterpret_cast<float*>(AG + r[k] * 8 + 4 + lane);
            const float4 o = a[(k + 1) % 3], q = a[(k + 2) % 3];
            asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(m * o.x * q.x),
                         "f"(m * o.y * q.y), "f"(m * o.z * q.z), "f"(m * o.w * q.w)
                         : "memory");
        }
    }
    if (acc == 1.2345f) *sink = acc;
}

// random 16-B loads with an explicit L2 prefetch-size qualifier (PF: 0 none, 64, 128, 256)
template <int PF>
__global__ void rand_load_pf(const uint4* __restrict__ a, uint64_t n, int64_t total, uint32_t* sink) {
    uint32_t acc = 0;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = tid; i < total; i += nt * 4) {
        uint4 v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint4* p = a + __umul64hi(mix(i + k * nt), n);
            if constexpr (PF == 64)
                asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w) : "l"(p));
            else if constexpr (PF == 128)
                asm volatile("ld.global.nc.L1::no_allocate.L2::128B.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w) : "l"(p));
            else if constexpr (PF == 1)
                asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w) : "l"(p));
            else
                v[k] = __ldg(p);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) acc += v[k].x ^ v[k].w;
    }
    if (acc == 0x12345678u) *sink = acc;
}

// TMA bulk reduction alternative to red.add.v4: each warp stages 8 rows of 64 B
// in shared memory and 8 lanes issue one cp.reduce.async.bulk (.add.f32) each
// into random rows of an L2-resident array (double-buffered per warp).
__global__ void bulk_red(float* G, uint64_t rows, int64_t total_rows) {
    __shared__ __align__(128) float4 buf[8][2][32];   // [warp][stage][lane]: 8 rows x 64 B
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    int stage = 0;
    for (int64_t i = gw * 8; i < total_rows; i += nw * 8) {
        if (lane < 8) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncwarp();
        buf[w][stage][lane] = make_float4(1.f, 1.f, 1.f, 1.f);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane < 8) {
            const uint64_t r = __umul64hi(mix(i + lane), rows);
            const unsigned sa = (unsigned)__cvta_generic_to_shared(&buf[w][stage][lane * 4]);
            asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 64;"
                         :: "l"(G + r * 16), "r"(sa) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        stage ^= 1;
    }
    if (lane < 8) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void copy4(const float4* __restrict__ a, float4* __restrict__ b, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}

template <typename F>
static float timeit(F f, int reps = 5) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t big = 2ull << 30, small = 2ull << 20;
    uint4* A;
    float4 *S, *B;
    uint32_t* sink;
    cudaMalloc(&A, big);
    cudaMalloc(&B, big);
    cudaMalloc(&S, small);
    cudaMalloc(&sink, 64);
    cudaMemset(A, 1, big);
    cudaMemset(S, 0, small);
    const int64_t total = 1ll << 26;
    printf("{");
    for (int blocks : {sms * 4, sms * 8, sms * 16}) {
        float ms = timeit([&] { rand_load<4><<<blocks, 256>>>(A, big / 16, total, 1, sink); });
        printf("\"rand16_hbm_b%d\": %.3e, ", blocks, total / (ms * 1e-3));
        ms = timeit([&] { rand_load<4><<<blocks, 256>>>(A, big / 32, total, 2, sink); });
        printf("\"rand32_hbm_b%d\": %.3e, ", blocks, total / (ms * 1e-3));
        ms = timeit([&] { rand_load<1><<<blocks, 256>>>(A, big / 16, total, 1, sink); });
        printf("\"rand16_hbm_ilp1_b%d\": %.3e, ", blocks, total / (ms * 1e-3));
        ms = timeit([&] { rand_rows<4><<<blocks, 256>>>(S, small / 64, total, (float*)sink); });
        printf("\"rand64_l2_rows_b%d\": %.3e, ", blocks, total / (ms * 1e-3));
        ms = timeit([&] { rand_red<<<blocks, 256>>>(S, small / 64, total); });
        printf("\"red64_l2_rows_b%d\": %.3e, ", blocks, total / (ms * 1e-3));
    }
    // contention: vector red into few rows (small modes of c1 / c3)
    for (int rows : {20, 1605, 4209, 10000}) {
        float ms = timeit([&] { rand_red<<<sms * 8, 256>>>(S, rows, total); });
        printf("\"red64_rows%d\": %.3e, ", rows, total / (ms * 1e-3));
    }
    // shared-memory scalar atomics into per-CTA rows
    cudaFuncSetAttribute(smem_red, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int srows : {20, 1605, 3000}) {
        for (int bps : {1, 2, 4}) {
            const size_t sb = (size_t)srows * 64;
            if (sb * bps > 200 * 1024) continue;
            float ms = timeit([&] { smem_red<<<sms * bps, 256, sb>>>((float*)sink, srows, total); });
            printf("\"smem_red64_rows%d_b%d\": %.3e, ", srows, bps, total / (ms * 1e-3));
        }
    }
    for (int blocks : {sms * 4, sms * 16}) {
        float ms = timeit([&] { rand_load_pf<0><<<blocks, 256>>>(A, big / 16, total, sink); });
        printf("\"rand16_pf0_b%d\": %.3e, ", blocks, total / (ms * 1e-3));
        ms = timeit([&] { rand_load_pf<1><<<blocks, 256>>>(A, big / 16, total, sink); });
        printf("\"rand16_noalloc_b%d\": %.3e, ", blocks, total / (ms * 1e-3));
        ms = timeit([&] { rand_load_pf<64><<<blocks, 256>>>(A, big / 16, total, sink); });
        printf("\"rand16_pf64_b%d\": %.3e, ", blocks, total / (ms * 1e-3));
        ms = timeit([&] { rand_load_pf<128><<<blocks, 256>>>(A, big / 16, total, sink); });
        printf("\"rand16_pf128_b%d\": %.3e, ", blocks, total / (ms * 1e-3));
    }
    for (int blocks : {sms * 2, sms * 4, sms * 8}) {
        float ms = timeit([&] { bulk_red<<<blocks, 256>>>((float*)S, small / 64, total); });
        printf("\"bulkred64_l2_rows_b%d\": %.3e, ", blocks, total / (ms * 1e-3));
    }
    // K2 skeleton on c2's shape: 30,000 rows of 64 B per array (A and G 1.9 MB), 2e7 samples
    {
        float4* G2;
        cudaMalloc(&G2, small);
        cudaMemset(G2, 0, small);
        const int64_t ns = 20000000;
        for (int wd : {0, 1}) {
            for (int blocks : {sms * 4, sms * 8}) {
                float ms = timeit([&] { k2_skeleton<<<blocks, 256>>>(A, big / 16, S, G2, 30000, ns, wd, (float*)sink); });
                printf("\"k2skel_dram%d_b%d_ms_per_2e7\": %.4f, ", wd, blocks, ms);
            }
        }
        cudaFree(G2);
    }
    // c4-shaped skeleton: 8.4M rows x 128 B (A|G interleaved, 1.07 GB), 2e7 samples
    {
        const uint64_t rows4 = 8400000;
        float4* AG;
        cudaMalloc(&AG, rows4 * 128);
        cudaMemset(AG, 0, rows4 * 128);
        for (int blocks : {sms * 4, sms * 8}) {
            float ms = timeit([&] { k2_skeleton_dram<<<blocks, 256>>>(A, big / 16, AG, rows4, 20000000, (float*)sink); });
            printf("\"k2skel_c4_b%d_ms_per_2e7\": %.4f, ", blocks, ms);
        }
        cudaFree(AG);
    }
    const int64_t n4 = big / 16;
    float ms = timeit([&] { copy4<<<sms * 8, 256>>>((const float4*)A, B, n4); });
    printf("\"copy_hbm_GBps\": %.1f}\n", 2.0 * big / (ms * 1e-3) / 1e9);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
