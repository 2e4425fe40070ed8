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

int main()
{
    long long *cyc, h[4] = {0, 0, 0, 0};
    double *sink;
    unsigned long long *words;
    cudaMalloc(&cyc, 4 * 8);
    cudaMalloc(&sink, 4 * NT * 8);
    cudaMalloc(&words, TB * 8);
    cudaMemset(words, 0, TB * 8);
    const int iters = 20000;
    pingpong<0><<<2, NT>>>(iters, cyc, sink);
    pingpong<1><<<2, NT>>>(iters, cyc, sink);
    pingpong<2><<<2, NT>>>(iters, cyc, sink);
    pingpong_l2<<<2, NT>>>(iters, cyc, words, sink);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("status %s\n", cudaGetErrorString(e));
    const char *nm[4] = {"DSMEM, 128 remote arrivals", "DSMEM, 4 warp arrivals + fence", "DSMEM bulk copy (1 KB)", "L2 flag-in-data words"};
    for (int i = 0; i < 4; ++i) printf("%-34s %6lld cycles per one-way hand-over (incl. __syncthreads)\n", nm[i], h[i]);
    return 0;
}
