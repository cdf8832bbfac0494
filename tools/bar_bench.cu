// Grid-barrier microbenchmark: cost per barrier of the persistent kernel's
// grid_sync variants at 148 / 296 / 592 CTAs of 256 threads (cooperative launch).
#include <cooperative_groups.h>
#include <cstdio>

namespace cg = cooperative_groups;

struct Bar {
    unsigned count;
    unsigned gen;
    unsigned sub[16 * 32];
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int V>
__device__ __forceinline__ void bar(Bar* b) {
    __syncthreads();
    if (threadIdx.x == 0) {
        if (V == 0 || V == 1) {
            volatile unsigned* genp = &b->gen;
            const unsigned gen = *genp;
            __threadfence();
            const unsigned arrived = atomicAdd(&b->count, 1u);
            if (arrived == gridDim.x - 1) {
                atomicExch(&b->count, 0u);
                __threadfence();
                atomicAdd(&b->gen, 1u);
            } else {
                while (*genp == gen)
                    if (V == 0) __nanosleep(32);
            }
            __threadfence();
        } else if (V == 2) {
            const unsigned gen = ld_acquire(&b->gen);
            const unsigned arrived = atom_add_acqrel(&b->count, 1u);
            if (arrived == gridDim.x - 1) {
                b->count = 0;
                st_release(&b->gen, gen + 1);
            } else {
                while (ld_acquire(&b->gen) == gen) {
                }
            }
        } else if (V == 3) {  // two-level arrival, 16 groups
            const unsigned gen = ld_acquire(&b->gen);
            const unsigned grp = blockIdx.x & 15;
            const unsigned gsize = (gridDim.x - grp + 15) / 16;
            const unsigned a = atom_add_acqrel(&b->sub[grp * 32], 1u);
            bool last = false;
            if (a == gsize - 1) {
                b->sub[grp * 32] = 0;
                const unsigned t = atom_add_acqrel(&b->count, 1u);
                if (t == 15) {
                    b->count = 0;
                    last = true;
                }
            }
            if (last) {
                st_release(&b->gen, gen + 1);
            } else {
                while (ld_acquire(&b->gen) == gen) {
                }
            }
        }
    }
    __syncthreads();
}

__device__ __forceinline__ void cluster_bar() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// V5: flip-bit barrier of the persistent kernel (one atomic per CTA).
// V6: cluster-hierarchical flip-bit: hardware cluster barrier, then one
// flip-bit atomic per cluster, then the cluster barrier again.
template <int V>
__device__ __forceinline__ void flipbar(Bar* b) {
    unsigned rank = 0, nunits = gridDim.x, unit = blockIdx.x;
    if (V == 6) {
        asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
        asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(nunits));
        asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(unit));
        cluster_bar();
    } else {
        __syncthreads();
    }
    if (rank == 0 && threadIdx.x == 0) {
        const unsigned inc = unit == 0 ? 0x80000000u - (nunits - 1u) : 1u;
        __threadfence();
        const unsigned old = atomicAdd(&b->count, inc);
        volatile unsigned* cnt = &b->count;
        while (((old ^ *cnt) & 0x80000000u) == 0u) {
        }
        __threadfence();
    }
    if (V == 6) cluster_bar();
    else __syncthreads();
}

__device__ __forceinline__ void red_release(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned atom_add_release(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

// V7: monotonic counter, posted (red.release) arrival, ld.acquire poll
// V8: the same with a relaxed poll and one fence.acq_rel after it
// V9: flip-bit with atom.add.release and an ld.acquire poll (no fences)
template <int V>
__device__ __forceinline__ void cntbar(Bar* b, unsigned& target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        if (V == 9) {
            const unsigned inc = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1u) : 1u;
            const unsigned old = atom_add_release(&b->count, inc);
            while (((old ^ ld_acquire(&b->count)) & 0x80000000u) == 0u) {
            }
        } else {
            target += gridDim.x;
            red_release(&b->count, 1u);
            if (V == 7) {
                while ((int)(ld_acquire(&b->count) - target) < 0) {
                }
            } else {
                while ((int)(ld_relaxed(&b->count) - target) < 0) {
                }
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            }
        }
    }
    __syncthreads();
}

template <int V>
__global__ void k(Bar* b, int n, unsigned long long* ns, float* sink) {
    unsigned target = 0;
    float acc = threadIdx.x;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < n; ++i) {
        acc = acc * 1.0001f + 1.f;
        if (V == 4) cg::this_grid().sync();
        else if (V >= 7) cntbar<V>(b, target);
        else if (V >= 5) flipbar<V>(b);
        else bar<V>(b);
    }
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (blockIdx.x == 0 && threadIdx.x == 0) *ns = t1 - t0;
    if (acc == 12345.f) *sink = acc;
}

template <int V>
void run(int nblocks, Bar* b, unsigned long long* ns, float* sink) {
    int n = 2000;
    void* args[] = {&b, &n, &ns, &sink};
    cudaMemset(b, 0, sizeof(Bar));
    cudaLaunchCooperativeKernel((const void*)k<V>, dim3(nblocks), dim3(256), args, 0, 0);
    cudaMemset(b, 0, sizeof(Bar));
    cudaLaunchCooperativeKernel((const void*)k<V>, dim3(nblocks), dim3(256), args, 0, 0);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h = 0;
    cudaMemcpy(&h, ns, 8, cudaMemcpyDeviceToHost);
    printf("variant %d blocks %4d: %s %.3f us/barrier\n", V, nblocks, cudaGetErrorString(e), h / 1e3 / n);
}

template <int V>
void runc(int nblocks, int cl, Bar* b, unsigned long long* ns, float* sink) {
    int n = 2000;
    cudaLaunchConfig_t c = {};
    c.gridDim = dim3(nblocks);
    c.blockDim = dim3(256);
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = cl;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    c.attrs = at;
    c.numAttrs = 2;
    cudaError_t e = cudaSuccess;
    for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(b, 0, sizeof(Bar));
        e = cudaLaunchKernelEx(&c, k<V>, b, n, ns, sink);
        if (e != cudaSuccess) break;
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    unsigned long long h = 0;
    cudaMemcpy(&h, ns, 8, cudaMemcpyDeviceToHost);
    printf("variant %d cluster %d blocks %4d: %s %.3f us/barrier\n", V, cl, nblocks, cudaGetErrorString(e),
           h / 1e3 / n);
    cudaGetLastError();
}

// V9 on a barrier word at a chosen offset of a large buffer (L2 slice / die)
__global__ void kaddr(unsigned* w, int n, unsigned long long* ns) {
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < n; ++i) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned inc = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1u) : 1u;
            const unsigned old = atom_add_release(w, inc);
            while (((old ^ ld_acquire(w)) & 0x80000000u) == 0u) {
            }
        }
        __syncthreads();
    }
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (blockIdx.x == 0 && threadIdx.x == 0) *ns = t1 - t0;
}

// V9 on the driver's cooperative-launch barrier word (CG: one cg grid sync first)
template <int CG>
__global__ void kws(int n, unsigned long long* ns, unsigned long long* addr) {
    unsigned long long t0, t1;
    if (CG == 1) cg::this_grid().sync();
    unsigned* w = &cg::details::get_grid_workspace()->barrier;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < n; ++i) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned inc = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1u) : 1u;
            const unsigned old = atom_add_release(w, inc);
            while (((old ^ ld_acquire(w)) & 0x80000000u) == 0u) {
            }
        }
        __syncthreads();
    }
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (blockIdx.x == 0 && threadIdx.x == 0) *ns = t1 - t0, *addr = (unsigned long long)w;
}

__device__ __forceinline__ unsigned ld_acquire_gen(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned atom_add_release_gen(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.add.release.gpu.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
// generic-address flip-bit (G bit 1: generic atom, bit 2: generic poll)
template <int G>
__global__ void kgen(unsigned* w, int n, unsigned long long* ns) {
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < n; ++i) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned inc = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1u) : 1u;
            const unsigned old = (G & 1) ? atom_add_release_gen(w, inc) : atom_add_release(w, inc);
            while (((old ^ ((G & 2) ? ld_acquire_gen(w) : ld_acquire(w))) & 0x80000000u) == 0u) {
            }
        }
        __syncthreads();
    }
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (blockIdx.x == 0 && threadIdx.x == 0) *ns = t1 - t0;
}
// flip-bit variants: S = nanosleep ns between polls (0: none), W: wait for the
// atomic's return before the first poll
template <int S, int W>
__global__ void kflip(unsigned* w, int n, unsigned long long* ns) {
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < n; ++i) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned inc = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1u) : 1u;
            unsigned old = atom_add_release(w, inc);
            if (W) old = __shfl_sync(1u, old, 0);
            while (((old ^ ld_acquire(w)) & 0x80000000u) == 0u) {
                if (S) __nanosleep(S);
            }
        }
        __syncthreads();
    }
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (blockIdx.x == 0 && threadIdx.x == 0) *ns = t1 - t0;
}
template <int S, int W>
void runflip(int nb, unsigned* w, unsigned long long* ns) {
    int n = 2000;
    void* args[] = {&w, &n, &ns};
    float best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(w, 0, 4);
        cudaLaunchCooperativeKernel((const void*)kflip<S, W>, dim3(nb), dim3(256), args, 0, 0);
        cudaDeviceSynchronize();
        unsigned long long h = 0;
        cudaMemcpy(&h, ns, 8, cudaMemcpyDeviceToHost);
        best = fminf(best, h / 1e3f / n);
    }
    printf("flip sleep %d wait %d blocks %d: %.3f us/barrier\n", S, W, nb, best);
}

template <int G>
void rungen(int nb, unsigned* w, unsigned long long* ns) {
    int n = 2000;
    void* args[] = {&w, &n, &ns};
    float best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(w, 0, 4);
        cudaLaunchCooperativeKernel((const void*)kgen<G>, dim3(nb), dim3(256), args, 0, 0);
        cudaDeviceSynchronize();
        unsigned long long h = 0;
        cudaMemcpy(&h, ns, 8, cudaMemcpyDeviceToHost);
        best = fminf(best, h / 1e3f / n);
    }
    printf("generic %d blocks %d: %.3f us/barrier\n", G, nb, best);
}

int main() {
    {
        unsigned* w;
        unsigned long long* ns4;
        cudaMalloc(&w, 4096);
        cudaMalloc(&ns4, 8);
        for (int nb : {148, 296, 592}) {
            runflip<0, 0>(nb, w, ns4);
            runflip<0, 1>(nb, w, ns4);
            runflip<32, 0>(nb, w, ns4);
            runflip<32, 1>(nb, w, ns4);
            runflip<100, 1>(nb, w, ns4);
            runflip<200, 1>(nb, w, ns4);
            runflip<500, 1>(nb, w, ns4);
        }
        for (int nb : {296, 592}) {
            rungen<0>(nb, w, ns4);
            rungen<1>(nb, w, ns4);
            rungen<2>(nb, w, ns4);
            rungen<3>(nb, w, ns4);
        }
    }
    {
        unsigned long long *ns3, *ad;
        cudaMalloc(&ns3, 8);
        cudaMalloc(&ad, 8);
        for (int nb : {296, 592}) {
            int n = 2000;
            void* args[] = {&n, &ns3, &ad};
            for (int rep = 0; rep < 6; ++rep) {
                cudaError_t e = cudaLaunchCooperativeKernel(rep & 1 ? (const void*)kws<1> : (const void*)kws<0>, dim3(nb), dim3(256), args, 0, 0);
                e = cudaDeviceSynchronize();
                unsigned long long h = 0, a = 0;
                cudaMemcpy(&h, ns3, 8, cudaMemcpyDeviceToHost);
                cudaMemcpy(&a, ad, 8, cudaMemcpyDeviceToHost);
                printf("driver-word cg-first %d blocks %d: %s %.3f us/barrier\n", rep & 1, nb, cudaGetErrorString(e), h / 1e3 / n); (void)a;
            }
        }
    }
    {
        unsigned* big;
        unsigned long long* ns2;
        cudaMalloc(&big, 64 << 20);
        cudaMalloc(&ns2, 8);
        for (int nb : {296, 592}) {
            for (long long off : {0LL, 32LL, 128LL, 4096LL, 65536LL, 1LL << 20, 3LL << 20, 5LL << 20, 7LL << 20, 11LL << 20, 13LL << 20, 17LL << 20, 33LL << 20}) {
                unsigned* w = big + off / 4;
                int n = 2000;
                void* args[] = {&w, &n, &ns2};
                float best = 1e9;
                for (int rep = 0; rep < 3; ++rep) {
                    cudaMemset(w, 0, 4);
                    cudaLaunchCooperativeKernel((const void*)kaddr, dim3(nb), dim3(256), args, 0, 0);
                    cudaDeviceSynchronize();
                    unsigned long long h = 0;
                    cudaMemcpy(&h, ns2, 8, cudaMemcpyDeviceToHost);
                    best = fminf(best, h / 1e3f / n);
                }
                printf("addr-offset %10lld blocks %d: %.3f us/barrier\n", off, nb, best);
            }
        }
    }
    Bar* b;
    unsigned long long* ns;
    float* sink;
    cudaMalloc(&b, sizeof(Bar));
    cudaMalloc(&ns, 8);
    cudaMalloc(&sink, 4);
    for (int nb : {148, 296, 592}) {
        run<0>(nb, b, ns, sink);
        run<1>(nb, b, ns, sink);
        run<2>(nb, b, ns, sink);
        run<3>(nb, b, ns, sink);
        run<4>(nb, b, ns, sink);
        run<5>(nb, b, ns, sink);
        run<7>(nb, b, ns, sink);
        run<8>(nb, b, ns, sink);
        run<9>(nb, b, ns, sink);
        for (int cl : {1, 2, 4, 8}) runc<5>(nb, cl, b, ns, sink);
        for (int cl : {2, 4, 8}) runc<6>(nb, cl, b, ns, sink);
    }
    return 0;
}
