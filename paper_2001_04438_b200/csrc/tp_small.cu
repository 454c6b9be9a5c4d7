// Small-batch kernel: Two-Pass softmax (Alg. 3) for a few rows of 1..3
// blocks (e.g. config 2: 64 x 32768), one cluster of 1..3 CTAs per row, the whole row staged
// in shared memory.
//
// The persistent kernels pay for their generality in latency (work queue, producer/consumer
// rings, grid- or cluster-wide row release); with fewer rows than SMs a cluster can simply own
// a row: thread 0 of each CTA starts one bulk copy per block it owns, the 16 warps run pass 1
// on each block as it lands, warp 0 forms the block values and stores them into every cluster
// CTA's shared memory, one cluster barrier, warp 0 forms the row statistics, pass 2 on the
// staged values (the row is read from HBM once).  Rows beyond the grid loop.
//
// Bit-identical to the other kernels: the same per-warp pass 1 (warp_pass1), block tree over
// the 16 warp pairs, canonical tree over the row's blocks (one group of nb <= 3 leaves, lane
// order) and pass 2.
#include "tp_ops.cuh"

namespace tp {

constexpr int kSmallMaxBlocks = 3;   // blocks staged per CTA
constexpr int kSmallMaxCluster = 3;  // CTAs per row

// One row per cluster of CL CTAs (CL = 1: a plain launch, every CTA its own cluster).  CTA q of
// the cluster stages and processes blocks q, q + CL, ... of the row (at most kSmallMaxBlocks);
// the block values go to every CTA of the cluster through distributed shared memory, one
// cluster barrier, and every CTA forms the same row statistics (the canonical tree over the
// row's blocks in lane order) for its pass 2.  Rows loop over the clusters.
template <typename In>
__global__ void __launch_bounds__(kThreads, 1) small_kernel(const KArgs a, int CL) {
    constexpr int V = InTraits<In>::V;
    extern __shared__ __align__(128) unsigned char dsm[];
    In* stages = reinterpret_cast<In*>(dsm);
    __shared__ __align__(8) uint64_t full_bar[kSmallMaxBlocks];
    __shared__ Pair wparts[kSmallMaxBlocks][kWarps];
    __shared__ unsigned char cbits[kSmallMaxBlocks][kWarps];
    __shared__ __align__(8) Pair rowvals[2][kSmallMaxBlocks * kSmallMaxCluster];  // by row parity
    __shared__ float2 s_st;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nb = (int)a.nb;
    const int q = (int)cluster_ctarank();
    const int nloc = (nb - q + CL - 1) / CL;  // this CTA's blocks: q + j * CL, j < nloc
    const In* x = static_cast<const In*>(a.x);
    if (threadIdx.x == 0) {
        for (int b = 0; b < kSmallMaxBlocks; ++b) mbar_init(&full_bar[b], 1);
        fence_mbar_init();
    }
    // every CTA of the cluster has started (and initialised its barriers) before any CTA
    // stores into a peer's shared memory (st.shared::cluster below)
    cluster_sync_all();
    pdl_wait_and_release();  // programmatic launch: set up above, touch memory only after the predecessor
    unsigned iter = 0;
    for (int64_t row = cluster_id_x(); row < a.rows; row += nclusters_x(), ++iter) {
        if (threadIdx.x == 0) {
            fence_proxy_async_smem();  // the previous row's reads of the stages come first
            for (int j = 0; j < nloc; ++j) {
                const int64_t e0 = (int64_t)(q + j * CL) * kBlockElems;
                const uint32_t bytes = (uint32_t)min((int64_t)kBlockElems, a.cols - e0) * (uint32_t)sizeof(In);
                mbar_arrive_expect_tx(&full_bar[j], bytes);
                tma_load_1d_nohint(stages + (size_t)j * kBlockElems, x + row * a.cols + e0, bytes, &full_bar[j]);
            }
        }
        for (int j = 0; j < nloc; ++j) {  // pass 1 per block as it lands
            mbar_wait_parity(&full_bar[j], iter & 1u);
            const int valid = (int)min((int64_t)kBlockElems, a.cols - (int64_t)(q + j * CL) * kBlockElems);
            BlockVals v;
            load_stage<In>(stages + (size_t)j * kBlockElems, v);
            Pair wp;
            const bool cl = warp_pass1<V>(v, valid, &wp);
            if (lane == 0) {
                wparts[j][warp] = wp;
                cbits[j][warp] = cl ? 1 : 0;
            }
        }
        __syncthreads();
        const int par = (int)(iter & 1u);
        if (warp == 0 && lane < nloc) {  // this CTA's block values into every cluster CTA
            const Pair bv = block_tree_warps(wparts[lane]);
            const uint32_t dst = smem_u32(&rowvals[par][q + lane * CL]);
            for (int r = 0; r < CL; ++r) st_cluster_f2(mapa(dst, (uint32_t)r), make_float2(bv.m, bv.n));
        }
        // all block values of the row everywhere; with double-buffered rowvals this barrier also
        // orders every CTA's reads of row k-1's values before anyone writes row k+1's
        cluster_sync_all();
        if (warp == 0) {  // row tree over the nb blocks (lane order), as every kernel
            const Pair bv = lane < nb ? rowvals[par][lane] : pair_identity();
            const Pair root = warp_tree_pairs(bv);
            if (lane == 0) s_st = make_float2(__fsub_rn(root.n, 1.0f), __fdiv_rn(0.5f, root.m));
        }
        __syncthreads();
        const float4 st = make_float4(s_st.x, s_st.y, 0.f, 0.f);
        for (int j = 0; j < nloc; ++j) {  // pass 2 on the staged blocks
            const int64_t e0 = (int64_t)(q + j * CL) * kBlockElems;
            const int valid = (int)min((int64_t)kBlockElems, a.cols - e0);
            BlockVals v;
            load_stage<In>(stages + (size_t)j * kBlockElems, v);
            op_pass2<V>(v, st, cbits[j][warp] != 0, a.y + row * a.cols + e0, valid, true);
        }
        __syncthreads();  // stages and parts free for the next row
    }
}

// The Three-Pass comparators on the same staging (Alg. 1 Recompute PAPER.md:88-104, Alg. 2
// Reload PAPER.md:108-128): max pass, exchange, Sum exp pass (Reload: also y = exp(x - mu)),
// exchange, output pass, all on the staged blocks except Reload's pass 3, which re-reads y from
// memory as the algorithm does.  Block and row reductions are the stream kernel's (bitwise).
template <typename In, int A>
__global__ void __launch_bounds__(kThreads, 1) small3_kernel(const KArgs a, int CL) {
    constexpr int V = InTraits<In>::V;
    extern __shared__ __align__(128) unsigned char dsm[];
    In* stages = reinterpret_cast<In*>(dsm);
    __shared__ __align__(8) uint64_t full_bar[kSmallMaxBlocks];
    __shared__ Part parts[kSmallMaxBlocks];
    __shared__ __align__(8) float2 rowvals[2][kSmallMaxBlocks * kSmallMaxCluster];  // by exchange parity
    __shared__ float4 s_st;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nb = (int)a.nb;
    const int q = (int)cluster_ctarank();
    const int nloc = (nb - q + CL - 1) / CL;
    const In* x = static_cast<const In*>(a.x);
    if (threadIdx.x == 0) {
        for (int b = 0; b < kSmallMaxBlocks; ++b) mbar_init(&full_bar[b], 1);
        fence_mbar_init();
    }
    // every CTA of the cluster has started (and initialised its barriers) before any CTA
    // stores into a peer's shared memory (st.shared::cluster below)
    cluster_sync_all();
    pdl_wait_and_release();
    unsigned iter = 0, xchg = 0;
    // block values (warp 0) -> every cluster CTA, cluster barrier, row value (warp 0) -> s_st
    auto exchange = [&](int phase) {
        const int par = (int)(xchg++ & 1u);
        if (warp == 0 && lane < nloc) {
            const Part& pt = parts[lane];
            float bv;
            if (phase == 0) {
                bv = pt.v[0].m;
                for (int w = 1; w < kWarps; ++w) bv = fmaxf(bv, pt.v[w].m);
            } else {
                float t[kWarps];
                for (int w = 0; w < kWarps; ++w) t[w] = pt.v[w].m;
                bv = block_tree_warps_sum(t);
            }
            const uint32_t dst = smem_u32(&rowvals[par][q + lane * CL]);
            for (int r = 0; r < CL; ++r) st_cluster_f2(mapa(dst, (uint32_t)r), make_float2(bv, 0.0f));
        }
        cluster_sync_all();
        if (warp == 0) {
            float root;
            if (phase == 0) root = warp_max(lane < nb ? rowvals[par][lane].x : -__int_as_float(0x7f800000));
            else root = warp_tree_sum(lane < nb ? rowvals[par][lane].x : 0.0f);
            if (lane == 0) s_st = row_stats_of<A>(phase, make_float2(root, 0.0f), s_st.x);
        }
        __syncthreads();
    };
    for (int64_t row = cluster_id_x(); row < a.rows; row += nclusters_x(), ++iter) {
        if (threadIdx.x == 0) {
            fence_proxy_async_smem();
            for (int j = 0; j < nloc; ++j) {
                const int64_t e0 = (int64_t)(q + j * CL) * kBlockElems;
                const uint32_t bytes = (uint32_t)min((int64_t)kBlockElems, a.cols - e0) * (uint32_t)sizeof(In);
                mbar_arrive_expect_tx(&full_bar[j], bytes);
                tma_load_1d_nohint(stages + (size_t)j * kBlockElems, x + row * a.cols + e0, bytes, &full_bar[j]);
            }
        }
        for (int j = 0; j < nloc; ++j) {  // pass 1: max
            mbar_wait_parity(&full_bar[j], iter & 1u);
            const int valid = (int)min((int64_t)kBlockElems, a.cols - (int64_t)(q + j * CL) * kBlockElems);
            BlockVals v;
            load_stage<In>(stages + (size_t)j * kBlockElems, v);
            op_max<V>(v, valid, parts[j]);
        }
        __syncthreads();
        exchange(0);
        const float mu = s_st.x;
        for (int j = 0; j < nloc; ++j) {  // pass 2: sum of exp(x - mu)
            const int64_t e0 = (int64_t)(q + j * CL) * kBlockElems;
            const int valid = (int)min((int64_t)kBlockElems, a.cols - e0);
            BlockVals v;
            load_stage<In>(stages + (size_t)j * kBlockElems, v);
            op_expsum<V, A == kReload>(v, valid, mu, parts[j], a.y + row * a.cols + e0, true);
        }
        __syncthreads();
        exchange(1);
        const float4 st = s_st;
        for (int j = 0; j < nloc; ++j) {  // pass 3: output
            const int64_t e0 = (int64_t)(q + j * CL) * kBlockElems;
            const int valid = (int)min((int64_t)kBlockElems, a.cols - e0);
            if (A == kRecompute) {
                BlockVals v;
                load_stage<In>(stages + (size_t)j * kBlockElems, v);
                op_out_recompute<V>(v, st, a.y + row * a.cols + e0, valid, true);
            } else {
                op_out_reload(st, a.y + row * a.cols + e0, valid, true);
            }
        }
        __syncthreads();
    }
}

// CTAs per row: as many as the row has blocks (<= 3) while the rows still fit one wave
static int small_cluster(int64_t rows, int64_t nb, int sms) {
    int CL = 1;
    while (CL < kSmallMaxCluster && CL < nb && rows * (CL + 1) <= sms) ++CL;
    if ((nb + CL - 1) / CL > kSmallMaxBlocks) return 0;
    return CL;
}

// rows of 1..3 blocks, aligned, no more rows than two waves of SMs: the latency regime
bool small_applies(int64_t rows, int64_t nb, int vec) {
    int dev = 0;
    cudaGetDevice(&dev);
    return vec && nb >= 1 && nb <= kSmallMaxBlocks && rows <= 2 * (int64_t)device_sms(dev);
}

template <typename In, int A>
cudaError_t launch_small(KArgs a, const LaunchOpts& o, cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    const int sms = device_sms(dev);
    int CL = small_cluster(a.rows, a.nb, sms);
    const int f = o.cluster_size;  // forced (tests, tuning) when it fits
    if (f >= 1 && f <= kSmallMaxCluster && f <= a.nb && (a.nb + f - 1) / f <= kSmallMaxBlocks) CL = f;
    if (CL < 1) return cudaErrorNotSupported;
    const int per = (int)((a.nb + CL - 1) / CL);
    const size_t dyn = (size_t)per * kBlockElems * sizeof(In);
    auto kern = A == kTwoPass ? small_kernel<In> : (A == kRecompute ? small3_kernel<In, kRecompute>
                                                                     : small3_kernel<In, kReload>);
    static DevCache configured[kMaxDevices];
    if (!configured[dev].load(std::memory_order_acquire)) {
        for (auto k : {small_kernel<In>, small3_kernel<In, kRecompute>, small3_kernel<In, kReload>})
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(kSmallMaxBlocks * kBlockElems * sizeof(In)));
        configured[dev].store(1, std::memory_order_release);
    }
    int64_t nclu = o.grid_ctas > 0 ? o.grid_ctas / CL : sms / CL;
    if (nclu < 1) nclu = 1;
    if (nclu > a.rows) nclu = a.rows;
    last_plan() = Plan{4, A, nclu * CL, CL, 0, (int)a.nb};
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(nclu * CL));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = dyn;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    // programmatic dependent launch: this grid may be scheduled while the previous kernel on
    // the stream runs (it waits for its completion before touching memory): the launch latency
    // of back-to-back short calls overlaps (development override TP_PDL=0)
    static const int pdl = dev_env_int("TP_PDL", 1);
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, kern, a, CL);
}

template cudaError_t launch_small<float, kTwoPass>(KArgs, const LaunchOpts&, cudaStream_t);
template cudaError_t launch_small<uint16_t, kTwoPass>(KArgs, const LaunchOpts&, cudaStream_t);
template cudaError_t launch_small<float, kRecompute>(KArgs, const LaunchOpts&, cudaStream_t);
template cudaError_t launch_small<uint16_t, kRecompute>(KArgs, const LaunchOpts&, cudaStream_t);
template cudaError_t launch_small<float, kReload>(KArgs, const LaunchOpts&, cudaStream_t);
template cudaError_t launch_small<uint16_t, kReload>(KArgs, const LaunchOpts&, cudaStream_t);

}  // namespace tp
