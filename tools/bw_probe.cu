// Bandwidth probe (tooling, not product): how fast can one B200 stream a
// 128 MB bf16 weight matrix through (a) plain 16-B LDG, (b) 1-D bulk async
// copies (cp.async.bulk) into a shared-memory ring, for different copy sizes,
// ring depths and CTAs per SM.  Consumers touch the data minimally (sum of
// one word per 16 B) so the copy engine / DRAM path is what is measured.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bw_probe tools/bw_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_ldg(const uint4* __restrict__ src, size_t n16, int* out) {
    uint32_t acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 7 * stride < n16; i += 8 * stride) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                         : "l"(src + i + u * stride));
#pragma unroll
        for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].w;
    }
    for (; i < n16; i += stride) acc ^= src[i].x;
    if (acc == 0x12345678) out[0] = 1;
}

// Each CTA streams chunks of `chunk` bytes (pieces of `piece` bytes each,
// one bulk copy per piece) through `stages` slots.
__global__ void k_bulk(const uint8_t* __restrict__ src, size_t total, int chunk, int piece,
                       int stages, int* out) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint64_t* full = (uint64_t*)(sm + (size_t)stages * chunk);
    uint64_t* empty = full + stages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwc = (blockDim.x >> 5) - 1;  // consumer warps
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&full[s])), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&empty[s])), "r"(nwc));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const size_t nchunks = total / chunk;
    if (warp == nwc) {
        if (lane) return;
        int q = 0;
        for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++q) {
            const int slot = q % stages;
            if (q >= stages) {
                const uint32_t par = ((q / stages) - 1) & 1;
                asm volatile("{\n\t.reg .pred p;\nW1_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W1_%=;\n}" ::"r"(su(&empty[slot])), "r"(par) : "memory");
            }
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[slot])), "r"(chunk) : "memory");
            for (int p = 0; p < chunk; p += piece)
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(su(sm + (size_t)slot * chunk + p)), "l"(src + c * chunk + p), "r"(piece), "r"(su(&full[slot])) : "memory");
        }
        return;
    }
    uint32_t acc = 0;
    int q = 0;
    for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++q) {
        const int slot = q % stages;
        const uint32_t par = (q / stages) & 1;
        asm volatile("{\n\t.reg .pred p;\nW2_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W2_%=;\n}" ::"r"(su(&full[slot])), "r"(par) : "memory");
        const uint4* s4 = (const uint4*)(sm + (size_t)slot * chunk);
        for (int i = warp * 32 + lane; i < chunk / 16; i += nwc * 32) acc ^= s4[i].x;
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[slot])) : "memory");
    }
    if (acc == 0x12345678) out[0] = 1;
}

int main() {
    const size_t bytes = 128ull << 20;
    uint8_t* buf;
    int* out;
    CK(cudaMalloc(&buf, bytes * 4));
    CK(cudaMalloc(&out, 4));
    CK(cudaMemset(buf, 1, bytes * 4));
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    // rotate over 4 buffers of 128 MB so L2 (126 MB) never holds the source
    auto timeit = [&](auto launch) {
        for (int w = 0; w < 3; ++w) launch(w & 3);
        cudaEventRecord(a);
        const int reps = 20;
        for (int r = 0; r < reps; ++r) launch(r & 3);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        return bytes * reps / (ms / 1e3) / 1e9;
    };
    for (int bpsm : {4, 8, 16}) {
        double gbs = timeit([&](int r) { k_ldg<<<sms * bpsm, 256>>>((const uint4*)(buf + r * bytes), bytes / 16, out); });
        printf("ldg  blocks/sm=%2d                                 %7.0f GB/s\n", bpsm, gbs);
    }
    for (int piece : {16384, 32768, 65536}) {
        for (int chunk : {16384, 32768, 65536}) {
            if (piece > chunk) continue;
            for (int stages : {4, 6}) {
                for (int cps : {1, 2, 3}) {
                    size_t smem = (size_t)stages * chunk + 2 * stages * 8;
                    if (smem * cps > 225 * 1024) continue;
                    cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                    double gbs = timeit([&](int r) {
                        k_bulk<<<sms * cps, 160, smem>>>(buf + r * bytes, bytes, chunk, piece, stages, out);
                    });
                    cudaError_t e = cudaGetLastError();
                    printf("bulk piece=%5d chunk=%5d stages=%d cta/sm=%d  %7.0f GB/s %s\n", piece, chunk,
                           stages, cps, gbs, e ? cudaGetErrorString(e) : "");
                }
            }
        }
    }
    return 0;
}
