// Hand-over latency of a 128-double block between two CTAs (development probe for the panel
// solve chain): ping-pong of ITERS round trips, per variant
//   0: DSMEM stores by 128 threads + 128 remote mbarrier arrivals (the panel's hand-over)
//   1: DSMEM stores + __syncwarp + one fence.acq_rel.cluster + remote arrive per warp (count 4)
//   2: local STS + named barrier + one cp.async.bulk shared::cta -> shared::cluster (complete_tx)
//   3: flag-in-data 64-bit words through global memory (L2), 128 pollers, no cluster
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 hop_bench.cu -o hop_bench
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

constexpr int TB = 128, NT = 512;
struct Sm {
    double y[TB];
    double stage[TB];
    unsigned long long mbar;
};

__device__ __forceinline__ void remote_arrive(unsigned long long *bar, unsigned rank)
{
    const unsigned la = (unsigned)__cvta_generic_to_shared(bar);
    unsigned ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(rank));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
__device__ __forceinline__ void wait_parity(unsigned long long *bar, unsigned par)
{
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    unsigned done = 0;
    while (!done)
        asm volatile("{\n .reg .pred P;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%1], %2;\n selp.u32 %0, 1, 0, P;\n}\n"
                     : "=r"(done) : "r"(a), "r"(par) : "memory");
}

template <int V>
__global__ void __cluster_dims__(2, 1, 1) pingpong(int iters, long long *cyc, double *sink)
{
    __shared__ Sm sm;
    cg::cluster_group cl = cg::this_cluster();
    const int rank = (int)cl.block_rank(), tid = threadIdx.x, lane = tid & 31;
    if (tid == 0) {
        const unsigned mb = (unsigned)__cvta_generic_to_shared(&sm.mbar);
        const int cnt = V == 0 ? TB : (V == 1 ? TB / 32 : 1);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mb), "r"(cnt) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < TB) sm.y[tid] = tid;
    cl.sync();
    Sm *peer = cl.map_shared_rank(&sm, rank ^ 1);
    unsigned par = 0;
    double v = tid;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const bool mine = (it & 1) == rank;  // whose turn to send
        if (mine) {
            if (V == 0 && tid < TB) {
                peer->y[tid] = v + it;
                remote_arrive(&sm.mbar, rank ^ 1);
            } else if (V == 1 && tid < TB) {
                peer->y[tid] = v + it;
                __syncwarp();
                if (lane == 0) {
                    asm volatile("fence.acq_rel.cluster;" ::: "memory");
                    remote_arrive(&sm.mbar, rank ^ 1);
                }
            } else if (V == 2) {
                if (tid < TB) sm.stage[tid] = v + it;
                asm volatile("bar.sync 1, %0;" ::"n"(TB) : "memory");  // tid < TB only (warps 0-3)
                if (tid == 0) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    const unsigned src = (unsigned)__cvta_generic_to_shared(sm.stage);
                    unsigned dst, mb;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(dst) : "r"((unsigned)__cvta_generic_to_shared(sm.y)), "r"(rank ^ 1));
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(mb) : "r"((unsigned)__cvta_generic_to_shared(&sm.mbar)), "r"(rank ^ 1));
                    asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(mb), "r"(TB * 8) : "memory");
                    asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                 ::"r"(dst), "r"(src), "r"(TB * 8), "r"(mb) : "memory");
                }
            }
        } else {
            wait_parity(&sm.mbar, par);
            par ^= 1u;
            if (tid < TB) v += sm.y[tid] * 1e-30;
        }
        __syncthreads();
    }
    const long long t1 = clock64();
    if (tid == 0 && rank == 0) cyc[V] = (t1 - t0) / iters;
    sink[blockIdx.x * NT + tid] = v;
}

__device__ __forceinline__ unsigned long long ldr(const unsigned long long *p)
{
    unsigned long long x;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(x) : "l"(p) : "memory");
    return x;
}
__device__ __forceinline__ void str(unsigned long long *p, unsigned long long x)
{
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(x) : "memory");
}
// V3: two CTAs (no cluster) exchange through global flag-in-data words
__global__ void pingpong_l2(int iters, long long *cyc, unsigned long long *words, double *sink)
{
    const int rank = blockIdx.x, tid = threadIdx.x;
    __shared__ double y[TB];
    double v = tid;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const bool mine = (it & 1) == rank;
        const unsigned ep = (unsigned)it + 1;
        if (mine) {
            if (tid < TB) str(words + tid, ((unsigned long long)ep << 32) | (unsigned)(tid + it));
        } else if (tid < TB) {
            unsigned long long w;
            do { w = ldr(words + tid); } while ((unsigned)(w >> 32) != ep);
            y[tid] = (double)(unsigned)w;
            v += y[tid] * 1e-30;
        }
        __syncthreads();
    }
    const long long t1 = clock64();
    if (tid == 0 && rank == 0) cyc[3] = (t1 - t0) / iters;
    sink[blockIdx.x * NT + tid] = v;
}

// V4: one 256-row hop of a 4-CTA cluster: register mat-vec (32 FMA per thread), fold of the 4
// column groups through shared memory, reduce-scatter of the 256-row partials over DSMEM
// (each CTA receives 3 x 64 partials, 192 remote arrivals per phase), sum, next hop
struct Sm4 {
    double part[4][256];
    double recv[3][64];
    double yslice[64];
    unsigned long long mbar;
};
__global__ void __cluster_dims__(4, 1, 1) hop4(int iters, long long *cyc, double *sink)
{
    __shared__ Sm4 sm;
    cg::cluster_group cl = cg::this_cluster();
    const int q = (int)cl.block_rank(), tid = threadIdx.x;
    if (tid == 0) {
        const unsigned mb = (unsigned)__cvta_generic_to_shared(&sm.mbar);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mb), "r"(192) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < 64) sm.yslice[tid] = 1.0 + tid * 1e-3;
    double tile[32];
    for (int i = 0; i < 32; ++i) tile[i] = 1e-3 * (tid + i);
    cl.sync();
    unsigned par = 0;
    const int rp = tid & 127, grp = tid >> 7;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        // (1) mat-vec: rows 2rp, 2rp+1 x 16 columns of this thread's group
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const double y = sm.yslice[grp * 16 + u];
            a0 = fma(tile[2 * u], y, a0);
            a1 = fma(tile[2 * u + 1], y, a1);
        }
        sm.part[grp][2 * rp] = a0;
        sm.part[grp][2 * rp + 1] = a1;
        __syncthreads();
        // (2) fold + (3) send the 3 foreign 64-row slices (threads 0..255: row r of 256)
        if (tid < 256) {
            const double v = (sm.part[0][tid] + sm.part[1][tid]) + (sm.part[2][tid] + sm.part[3][tid]);
            const int dst = tid >> 6;
            if (dst != q) {
                Sm4 *peer = cl.map_shared_rank(&sm, dst);
                const int slot = q < dst ? q : q - 1;
                peer->recv[slot][tid & 63] = v;
                remote_arrive(&sm.mbar, dst);
            } else {
                sm.part[0][tid] = v;  // own slice
            }
        }
        // (4) wait for the 3 peers, sum the own slice -> next hop's y slice
        wait_parity(&sm.mbar, par);
        par ^= 1u;
        if (tid < 64) sm.yslice[tid] = sm.part[0][64 * q + tid] + (sm.recv[0][tid] + sm.recv[1][tid] + sm.recv[2][tid]) * 1e-30;
        __syncthreads();
    }
    const long long t1 = clock64();
    if (tid == 0 && q == 0) cyc[0] = (t1 - t0) / iters;
    sink[blockIdx.x * 512 + tid] = sm.yslice[tid & 63];
    cl.sync();
}

int main()
{
    long long *cyc, h[4] = {0, 0, 0, 0};
    double *sink;
    unsigned long long *words;
    cudaMalloc(&cyc, 4 * 8);
    cudaMalloc(&sink, 8 * NT * 8);
    cudaMalloc(&words, TB * 8);
    cudaMemset(words, 0, TB * 8);
    const int iters = 20000;
    pingpong<0><<<2, NT>>>(iters, cyc, sink);
    pingpong<1><<<2, NT>>>(iters, cyc, sink);
    pingpong<2><<<2, NT>>>(iters, cyc, sink);
    pingpong_l2<<<2, NT>>>(iters, cyc, words, sink);
    long long *c4;
    cudaMalloc(&c4, 8);
    hop4<<<4, NT>>>(iters, c4, sink);
    cudaError_t e = cudaDeviceSynchronize();
    long long h4 = 0;
    cudaMemcpy(&h4, c4, 8, cudaMemcpyDeviceToHost);
    printf("4-CTA 256-row hop (mat-vec + fold + DSMEM reduce-scatter + sum): %lld cycles\n", h4);
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("status %s\n", cudaGetErrorString(e));
    const char *nm[4] = {"DSMEM, 128 remote arrivals", "DSMEM, 4 warp arrivals + fence", "DSMEM bulk copy (1 KB)", "L2 flag-in-data words"};
    for (int i = 0; i < 4; ++i) printf("%-34s %6lld cycles per one-way hand-over (incl. __syncthreads)\n", nm[i], h[i]);
    return 0;
}
