// Small-batch kernel: Two-Pass softmax (Alg. 3) for a few rows of 1..3
// blocks (e.g. config 2: 64 x 32768), one CTA per row, the whole row staged in shared memory.
//
// The persistent kernels pay for their generality in latency (work queue, producer/consumer
// rings, grid- or cluster-wide row release); with fewer rows than SMs a CTA can simply own a
// row: thread 0 starts one bulk copy per block, the 16 warps run pass 1 on each block as it
// lands, one barrier, warp 0 forms the block values and the row statistics, one barrier, pass 2
// on the staged values (the row is read from HBM once).  Rows beyond the grid loop.
//
// Bit-identical to the other kernels: the same per-warp pass 1 (warp_pass1), block tree over
// the 16 warp pairs, canonical tree over the row's blocks (one group of nb <= 3 leaves, lane
// order) and pass 2.
#include "tp_ops.cuh"

namespace tp {

constexpr int kSmallMaxBlocks = 3;

template <typename In>
__global__ void __launch_bounds__(kThreads, 1) small_kernel(const KArgs a) {
    constexpr int V = InTraits<In>::V;
    extern __shared__ __align__(128) unsigned char dsm[];
    In* stages = reinterpret_cast<In*>(dsm);
    __shared__ __align__(8) uint64_t full_bar[kSmallMaxBlocks];
    __shared__ Pair wparts[kSmallMaxBlocks][kWarps];
    __shared__ unsigned char cbits[kSmallMaxBlocks][kWarps];
    __shared__ float2 s_st;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nb = (int)a.nb;
    const In* x = static_cast<const In*>(a.x);
    if (threadIdx.x == 0) {
        for (int b = 0; b < kSmallMaxBlocks; ++b) mbar_init(&full_bar[b], 1);
        fence_mbar_init();
    }
    __syncthreads();
    unsigned iter = 0;
    for (int64_t row = blockIdx.x; row < a.rows; row += gridDim.x, ++iter) {
        if (threadIdx.x == 0) {
            fence_proxy_async_smem();  // the previous row's reads of the stages come first
            for (int b = 0; b < nb; ++b) {
                const int64_t e0 = (int64_t)b * kBlockElems;
                const uint32_t bytes = (uint32_t)min((int64_t)kBlockElems, a.cols - e0) * (uint32_t)sizeof(In);
                mbar_arrive_expect_tx(&full_bar[b], bytes);
                tma_load_1d_nohint(stages + (size_t)b * kBlockElems, x + row * a.cols + e0, bytes, &full_bar[b]);
            }
        }
        for (int b = 0; b < nb; ++b) {  // pass 1 per block as it lands
            mbar_wait_parity(&full_bar[b], iter & 1u);
            const int valid = (int)min((int64_t)kBlockElems, a.cols - (int64_t)b * kBlockElems);
            BlockVals v;
            load_stage<In>(stages + (size_t)b * kBlockElems, v);
            Pair wp;
            const bool cl = warp_pass1<V>(v, valid, &wp);
            if (lane == 0) {
                wparts[b][warp] = wp;
                cbits[b][warp] = cl ? 1 : 0;
            }
        }
        __syncthreads();
        if (warp == 0) {  // block values, then the row tree over the nb blocks (lane order)
            Pair bv = pair_identity();
            if (lane < nb) bv = block_tree_warps(wparts[lane]);
            const Pair root = warp_tree_pairs(bv);
            if (lane == 0) s_st = make_float2(__fsub_rn(root.n, 1.0f), __fdiv_rn(0.5f, root.m));
        }
        __syncthreads();
        const float4 st = make_float4(s_st.x, s_st.y, 0.f, 0.f);
        for (int b = 0; b < nb; ++b) {  // pass 2 on the staged row
            const int valid = (int)min((int64_t)kBlockElems, a.cols - (int64_t)b * kBlockElems);
            BlockVals v;
            load_stage<In>(stages + (size_t)b * kBlockElems, v);
            op_pass2<V>(v, st, cbits[b][warp] != 0, a.y + row * a.cols + (int64_t)b * kBlockElems, valid, true);
        }
        __syncthreads();  // stages and parts free for the next row
    }
}

// rows of 1..3 blocks, aligned, no more rows than two waves of SMs: the latency regime
bool small_applies(int64_t rows, int64_t nb, int vec) {
    int dev = 0;
    cudaGetDevice(&dev);
    return vec && nb >= 1 && nb <= kSmallMaxBlocks && rows <= 2 * (int64_t)device_sms(dev);
}

template <typename In>
cudaError_t launch_small(KArgs a, const LaunchOpts& o, cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    const size_t dyn = (size_t)a.nb * kBlockElems * sizeof(In);
    static int configured[64];
    if (!configured[dev]) {
        cudaFuncSetAttribute(small_kernel<In>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(kSmallMaxBlocks * kBlockElems * sizeof(In)));
        configured[dev] = 1;
    }
    int64_t grid = o.grid_ctas > 0 ? o.grid_ctas : device_sms(dev);
    if (grid > a.rows) grid = a.rows;
    last_plan() = Plan{4, kTwoPass, grid, 0, 0, (int)a.nb};
    small_kernel<In><<<(unsigned)grid, kThreads, dyn, s>>>(a);
    return cudaGetLastError();
}

template cudaError_t launch_small<float>(KArgs, const LaunchOpts&, cudaStream_t);
template cudaError_t launch_small<uint16_t>(KArgs, const LaunchOpts&, cudaStream_t);

}  // namespace tp
