// nvlsbench.cu -- NVLink / NVLS ceilings for the access patterns of the fused
// exchange (fused.cu) on N GPUs of one node, one process (development tool; not
// part of libgcp.so).  Every GPU owns a 1/N shard of an S-byte symmetric window
// and, over its shard:
//   peer_read  : loads the shard from all N windows (unicast NVLink) and sums
//   mm_reduce  : one multimem.ld_reduce.add.v4.f32 per vector (NVLS, switch sum)
//   peer_store : stores the shard into all N windows (unicast)
//   mm_store   : one multimem.st.v4.f32 per vector (NVLS broadcast)
//   local_rw   : reads + writes its shard locally (HBM reference)
// for U vectors in flight per thread and C CTAs (256 threads) per SM.  Prints
// one JSON line: GB/s of shard bytes per GPU (max time over GPUs).
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/nvlsbench tools/nvlsbench.cu \
//      -I$NCCL/include -L$NCCL/lib -l:libnccl.so.2 -Xlinker -rpath=$NCCL/lib
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));     \
            exit(1);                                                                       \
        }                                                                                  \
    } while (0)
#define NK(x)                                                                              \
    do {                                                                                   \
        ncclResult_t r_ = (x);                                                             \
        if (r_ != ncclSuccess) {                                                           \
            fprintf(stderr, "%s:%d nccl %s\n", __FILE__, __LINE__, ncclGetErrorString(r_)); \
            exit(1);                                                                       \
        }                                                                                  \
    } while (0)

enum { PEER_READ = 0, MM_REDUCE = 1, PEER_STORE = 2, MM_STORE = 3, LOCAL_RW = 4 };
static const char* kNames[] = {"peer_read", "mm_reduce", "peer_store", "mm_store", "local_rw"};

template <int MODE, int U>
__global__ void __launch_bounds__(256) k_bench(ncclDevComm comm, ncclWindow_t win, float4* out, int64_t shard_vecs,
                                               int64_t first_vec, int nranks) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v0 = tid; v0 < shard_vecs; v0 += nt * U) {
        float4 acc[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
            const int64_t v = v0 + (int64_t)u * nt;
            if (v >= shard_vecs) continue;
            const size_t ob = (size_t)(first_vec + v) * 16;
            if constexpr (MODE == PEER_READ) {
                for (int r = 0; r < nranks; ++r) {
                    const float4 x = *reinterpret_cast<const float4*>(ncclGetLsaPointer(win, ob, r));
                    acc[u].x += x.x; acc[u].y += x.y; acc[u].z += x.z; acc[u].w += x.w;
                }
            } else if constexpr (MODE == MM_REDUCE) {
                const float* p = static_cast<const float*>(ncclGetLsaMultimemPointer(win, ob, comm));
                asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                             : "=f"(acc[u].x), "=f"(acc[u].y), "=f"(acc[u].z), "=f"(acc[u].w)
                             : "l"(p)
                             : "memory");
            } else if constexpr (MODE == LOCAL_RW) {
                acc[u] = *reinterpret_cast<const float4*>(ncclGetLocalPointer(win, ob));
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t v = v0 + (int64_t)u * nt;
            if (v >= shard_vecs) continue;
            const size_t ob = (size_t)(first_vec + v) * 16;
            const float4 val = make_float4(1.f, 2.f, 3.f, (float)u);
            if constexpr (MODE == PEER_STORE) {
                for (int r = 0; r < nranks; ++r) *reinterpret_cast<float4*>(ncclGetLsaPointer(win, ob, r)) = val;
            } else if constexpr (MODE == MM_STORE) {
                float* p = static_cast<float*>(ncclGetLsaMultimemPointer(win, ob, comm));
                asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(val.x),
                             "f"(val.y), "f"(val.z), "f"(val.w)
                             : "memory");
            } else {
                out[v] = acc[u];   // keeps the loads live; local write
            }
        }
    }
}

template <int MODE>
static void launch(int U, int grid, cudaStream_t s, ncclDevComm dc, ncclWindow_t w, float4* out, int64_t sv,
                   int64_t fv, int n) {
    switch (U) {
        case 1: k_bench<MODE, 1><<<grid, 256, 0, s>>>(dc, w, out, sv, fv, n); break;
        case 2: k_bench<MODE, 2><<<grid, 256, 0, s>>>(dc, w, out, sv, fv, n); break;
        case 4: k_bench<MODE, 4><<<grid, 256, 0, s>>>(dc, w, out, sv, fv, n); break;
        default: k_bench<MODE, 8><<<grid, 256, 0, s>>>(dc, w, out, sv, fv, n); break;
    }
}

static void launch_mode(int mode, int U, int grid, cudaStream_t s, ncclDevComm dc, ncclWindow_t w, float4* out,
                        int64_t sv, int64_t fv, int n) {
    switch (mode) {
        case PEER_READ: launch<PEER_READ>(U, grid, s, dc, w, out, sv, fv, n); break;
        case MM_REDUCE: launch<MM_REDUCE>(U, grid, s, dc, w, out, sv, fv, n); break;
        case PEER_STORE: launch<PEER_STORE>(U, grid, s, dc, w, out, sv, fv, n); break;
        case MM_STORE: launch<MM_STORE>(U, grid, s, dc, w, out, sv, fv, n); break;
        default: launch<LOCAL_RW>(U, grid, s, dc, w, out, sv, fv, n); break;
    }
}

int main(int argc, char** argv) {
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    const size_t S = (argc > 1 ? atol(argv[1]) : 228) << 20;   // window bytes (MB)
    std::vector<int> devs(n);
    for (int i = 0; i < n; ++i) devs[i] = i;
    std::vector<ncclComm_t> comms(n);
    NK(ncclCommInitAll(comms.data(), n, devs.data()));
    std::vector<void*> buf(n);
    std::vector<float4*> out(n);
    std::vector<ncclWindow_t> win(n);
    std::vector<ncclDevComm> dc(n);
    std::vector<cudaStream_t> st(n);
    std::vector<cudaEvent_t> e0(n), e1(n);
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    for (int i = 0; i < n; ++i) {
        CK(cudaSetDevice(i));
        NK(ncclMemAlloc(&buf[i], S));
        CK(cudaMemset(buf[i], 0, S));
        CK(cudaMalloc(&out[i], S / n + 4096));
        CK(cudaStreamCreate(&st[i]));
        CK(cudaEventCreate(&e0[i]));
        CK(cudaEventCreate(&e1[i]));
    }
    bool mm = true;
    {
        ncclDevCommRequirements reqs;
        memset(&reqs, 0, sizeof(reqs));
        reqs.lsaMultimem = true;
        NK(ncclGroupStart());
        for (int i = 0; i < n; ++i) {
            CK(cudaSetDevice(i));
            NK(ncclCommWindowRegister(comms[i], buf[i], S, &win[i], NCCL_WIN_COLL_SYMMETRIC));
        }
        NK(ncclGroupEnd());
        NK(ncclGroupStart());
        for (int i = 0; i < n; ++i) {
            CK(cudaSetDevice(i));
            NK(ncclDevCommCreate(comms[i], &reqs, &dc[i]));
        }
        NK(ncclGroupEnd());
        for (int i = 0; i < n; ++i) mm = mm && dc[i].lsaMultimem.mcBasePtr != nullptr;
    }
    const int64_t vecs = (int64_t)(S / 16);
    const int64_t sv = vecs / n;
    printf("{\"gpus\": %d, \"window_MB\": %zu, \"multimem\": %s", n, S >> 20, mm ? "true" : "false");
    for (int mode = 0; mode < 5; ++mode) {
        if (!mm && (mode == MM_REDUCE || mode == MM_STORE)) continue;
        for (int cps : {1, 2, 4, 8}) {
            for (int U : {1, 2, 4, 8}) {
                float best = 1e30f;
                for (int rep = 0; rep < 4; ++rep) {
                    for (int i = 0; i < n; ++i) { CK(cudaSetDevice(i)); CK(cudaDeviceSynchronize()); }
                    for (int i = 0; i < n; ++i) {
                        CK(cudaSetDevice(i));
                        CK(cudaEventRecord(e0[i], st[i]));
                        launch_mode(mode, U, sms * cps, st[i], dc[i], win[i], out[i], sv, sv * i, n);
                        CK(cudaEventRecord(e1[i], st[i]));
                    }
                    float mx = 0.f;
                    for (int i = 0; i < n; ++i) {
                        CK(cudaSetDevice(i));
                        CK(cudaEventSynchronize(e1[i]));
                        float ms;
                        CK(cudaEventElapsedTime(&ms, e0[i], e1[i]));
                        mx = ms > mx ? ms : mx;
                    }
                    if (rep > 0 && mx < best) best = mx;   // rep 0 warms up
                }
                printf(", \"%s_c%d_u%d\": %.1f", kNames[mode], cps, U, (double)sv * 16 / (best * 1e-3) / 1e9);
            }
        }
    }
    printf("}\n");
    for (int i = 0; i < n; ++i) {
        CK(cudaSetDevice(i));
        CK(cudaDeviceSynchronize());
    }
    return 0;
}
