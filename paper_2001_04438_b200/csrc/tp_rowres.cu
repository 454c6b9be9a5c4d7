// Resident-row kernel: Two-Pass softmax (Alg. 3) for rows of 4..64 blocks split
// over a group of G CTAs whose shares of two consecutive rows fit shared memory (bf16: up to 3
// blocks per CTA and row, fp32: 1), e.g. config 4 (256 x 800,000 = 49 blocks per row).
//
// Why: the cluster kernel (tp_rowcl.cu) runs pass 1 of row k and pass 2 of row k-1 on the same
// SM at once with two teams of 8 warps; measured, the two passes then share the SM at ~1.65 us per
// block-pass against ~1.0 us for 16 warps on one pass alone, and pass 2's re-reads miss L2 (bf16:
// about half of them; a row period is a whole L2 footprint).  Here every CTA stages its share of
// a row once and keeps it until pass 2: the row is read from HBM once, and all 16 warps run one
// pass at a time (pass 1 of row k+1, then pass 2 of row k).  A group is any G CTAs of the grid,
// not one GPC (8-CTA clusters fit only 15 x 8 SMs): its CTAs exchange block values through the
// workspace.  A first version with one staged row per CTA and CTA barriers around the exchange
// measured 392 us on C4 bf16 (cluster kernel 350 us on the same box): every group ran pass 1,
// the exchange and pass 2 in lockstep, so DRAM idled during pass 1 and was oversubscribed by
// pass 2's stores; with two rows staged the exchange hides behind the next row's pass 1 and
// the passes alternate at block granularity.
//
// Bit-identical to the other kernels: the same per-warp pass 1 (warp_pass1, clamp decision per
// warp), block tree over the 16 warp values, canonical tree over the row's blocks (one group of
// nb <= 64 leaves, warp_tree64 as tp_rowcl.cu's cl_row_stats) and pass 2 (op_pass2).
//
// Group exchange (global memory, workspace control region `res_vals`): each block value is
// stored as two 64-bit words, bits(m) and bits(n), each with the launch's tag (workspace epoch +
// 1) in its upper half; a CTA's statistics warp loads the row's nb slots until every word carries
// the tag (single-copy-atomic 64-bit accesses: a tagged word is a complete value), then forms the
// row statistics.  The first version released each value by a row ticket (red.release) and
// polled the ticket: two round trips to L2 per row under full HBM load instead of one
// (C4 bf16 ~300 us).  The last CTA out advances the epoch; the control region (tags included)
// is zeroed whenever a workspace changes shape, which also resets the epoch.  All CTAs of a
// launch must be co-resident (one per SM, grid <= SMs), as for the persistent kernels; a wait
// that exceeds kWaitTimeoutNs aborts the launch (watchdog, TP_EWATCHDOG on the next call)
// instead of hanging the GPU.
#include "tp_rowres.cuh"

#ifndef TP_RES_UNROLL
#define TP_RES_UNROLL 1
#endif
#ifndef TP_RES_FUSE
#define TP_RES_FUSE 1
#endif
#ifndef TP_RES_EXP
#define TP_RES_EXP 0  // development timing experiments (wrong outputs for 2, 4, 8): never set in a release build
#endif

namespace tp {

constexpr bool kResFuse = TP_RES_FUSE != 0;
constexpr int kResUnroll = TP_RES_UNROLL;

// Roles.  16 compute warps: pass 1 of rows 0 .. ahead-1; then per row k: pass 1 of row k+ahead,
// pass 2 of row k (each warp arrives on a block's p1_bar after pass 1 and on its empty_bar after
// reading the stage in pass 2).  Four service warps, none of which stores outputs (a release
// then waits only for its own block value, not for a queue of streaming stores), each blocking
// only on its own waits so that their latencies overlap: the post warp (block value = tree over
// the 16 warp values, stored as tagged words), two statistics warps (even / odd
// rows: wait for the group's nb tagged values, canonical tree, s_st + stats_bar), the load warp (stages rows in; refills a stage with the row
// nbuf ahead once pass 2 has read it).  20 warps: the same 96-register cap as 17.


// 8 consecutive values of this thread (group g of pass1_thread: BlockVals v[8 g .. 8 g + 7]) from a staged block.
template <typename In>
__device__ __forceinline__ void load_group8(const In* stage, int g, float (&x)[8]) {
    constexpr int V = InTraits<In>::V;
    if constexpr (V == 8) {
        unpack_bf16x8(*reinterpret_cast<const uint4*>(stage + vec_off<8>((int)threadIdx.x, g)), x);
    } else {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float4 a = *reinterpret_cast<const float4*>(stage + vec_off<4>((int)threadIdx.x, 2 * g + h));
            x[4 * h] = a.x; x[4 * h + 1] = a.y; x[4 * h + 2] = a.z; x[4 * h + 3] = a.w;
        }
    }
}

// Pass 2 of one whole, unclamped staged block (s2 -> yb) and pass 1 of another (s1), interleaved 8
// elements at a time in one instruction stream: pass 2's stores leave the SM at the pace of both
// passes' arithmetic instead of in a burst per block (the SM's store path takes ~31 B/clk, less
// than pass 2 alone produces), and each pass's dependent chains fill the other's latencies.
// Exactly pass1_thread<V, true, false> and pass2_store_full<V, false>: the same operations on the
// same values in the same per-thread order.  Returns the unclamped thread pair of s1.
template <typename In>
__device__ __forceinline__ Pair fused_pass1_pass2(const In* s1, const In* s2, float4 st, float* yb) {
    constexpr int V = InTraits<In>::V;
    const Pass2Consts k = pass2_consts(st.x, st.y);
    AccV acc = accv_init();
#pragma unroll kResUnroll  // one basic block per group: ptxas otherwise schedules every store of the block after the arithmetic
    for (int g = 0; g < kPerThread / 8; ++g) {
        float x2[8], x1[8], o[8];
        load_group8<In>(s2, g, x2);
        load_group8<In>(s1, g, x1);
#pragma unroll
        for (int q = 0; q < 8; q += 2) {
            const float2 y = pass2_pair<false>(make_float2(x2[q], x2[q + 1]), k);
            o[q] = y.x;
            o[q + 1] = y.y;
        }
#pragma unroll
        for (int h = 0; h < 8; h += 4)
            // volatile: issued here, between the groups (the compiler otherwise sinks a block's stores to the end)
            asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(yb + vec_off<V>((int)threadIdx.x, (8 / V) * g + h / V) + (h % V)),
                         "f"(o[h]), "f"(o[h + 1]), "f"(o[h + 2]), "f"(o[h + 3])
                         : "memory");
        float2 m[4], v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) ext_exp2v<false>(make_float2(x1[2 * j], x1[2 * j + 1]), m[j], v[j]);
        acc_add8v(acc, m, v);
    }
    return accv_pair(acc);
}

template <typename In>
__global__ void __launch_bounds__(kResThreads, 1) rowres_kernel(const KArgs a, int G, int ngroups, int nbuf, int ahead) {
    constexpr int V = InTraits<In>::V;
    constexpr int S = kResSlots;
    extern __shared__ __align__(128) unsigned char dsm[];
    In* stages = reinterpret_cast<In*>(dsm);  // [nbuf][nloc] blocks; slot index b * nloc + j
    __shared__ __align__(8) uint64_t full_bar[S];
    __shared__ __align__(8) uint64_t p1_bar[S];
    __shared__ __align__(8) uint64_t empty_bar[S];
    __shared__ __align__(8) uint64_t stats_bar[S];
    __shared__ Pair wparts[S][kWarps];
    __shared__ unsigned char cbits[S][kWarps];
    __shared__ float2 s_st[S];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nb = (int)a.nb;
    const int grp = (int)blockIdx.x / G;
    const int q = (int)blockIdx.x - grp * G;
    const int nloc = (nb - q + G - 1) / G;  // this CTA's blocks: q + j * G, j < nloc
    WsHeader* hdr = reinterpret_cast<WsHeader*>(a.ws);
    unsigned* err = &hdr->error;
    if (grp >= ngroups) return;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full_bar[i], 1);
            mbar_init(&p1_bar[i], kWarps);
            mbar_init(&empty_bar[i], kWarps);
            mbar_init(&stats_bar[i], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    pdl_wait_and_release();  // programmatic launch: touch memory only after the predecessor
    publish_abort_word(a);
    __shared__ unsigned s_epoch;
    if (threadIdx.x == 0) s_epoch = *reinterpret_cast<volatile unsigned*>(&hdr->epoch);
    __syncthreads();
    const unsigned long long tag = (unsigned long long)(s_epoch + 1u) << 32;  // this launch's tag
    const int64_t nrows = (a.rows - grp + ngroups - 1) / ngroups;  // the group's rows: grp + k ngroups
    const ResDiv ring(nbuf);
    auto slot = [&](int64_t k, int j) { return stages + ((size_t)ring.rem(k) * nloc + j) * kBlockElems; };
    auto ph = [&](int64_t k) { return (uint32_t)(ring.quot(k) & 1); };  // phase parity of row k's use
    // block value slots: (bits(m) | tag, bits(n) | tag), two single-copy-atomic 64-bit words
    unsigned long long* slots = reinterpret_cast<unsigned long long*>(a.ws + a.lay.res_vals);

    auto load_role = [&]() {  // ------------------------------------------------------ load warp
        if (lane == 0) {
            const In* x = static_cast<const In*>(a.x);
            const uint64_t pol = policy_evict_first();  // every byte is read from HBM once
            auto stage_in = [&](int64_t k, int j) {
                const int64_t row = grp + k * ngroups;
                const int64_t e0 = (int64_t)(q + j * G) * kBlockElems;
                const uint32_t bytes = (uint32_t)min((int64_t)kBlockElems, a.cols - e0) * (uint32_t)sizeof(In);
                uint64_t* fb = &full_bar[ring.rem(k) * nloc + j];
                mbar_arrive_expect_tx(fb, bytes);
                tma_load_1d(slot(k, j), x + row * a.cols + e0, bytes, fb, pol);
            };
            for (int64_t k = 0; k < nbuf && k < nrows; ++k)
                for (int j = 0; j < nloc; ++j) stage_in(k, j);
            for (int64_t k = 0; k + nbuf < nrows; ++k)
                for (int j = 0; j < nloc; ++j) {  // pass 2 of row k has read the stage
                    if (!((TP_RES_EXP & 1) ? wait_sleep_or_abort(&empty_bar[ring.rem(k) * nloc + j], ph(k), err, 2u)
                                           : wait_or_abort(&empty_bar[ring.rem(k) * nloc + j], ph(k), err, 2u))) return;
                    fence_proxy_async_smem();
                    stage_in(k + nbuf, j);
                }
        }
    };
    auto post_role = [&]() {  // ------------------------------------------------------ post warp
        for (int64_t k = 0; k < nrows; ++k) {
            const int b = ring.rem(k);
            const int64_t row = grp + k * ngroups;
            for (int j = 0; j < nloc; ++j) {
                if (!((TP_RES_EXP & 1) ? wait_sleep_or_abort(&p1_bar[b * nloc + j], ph(k), err, 32u)
                                       : wait_or_abort(&p1_bar[b * nloc + j], ph(k), err, 32u))) return;
                // block value: perfect tree over the 16 warp values in warp order (lanes 16-31
                // identities: merge(v, identity) == v), as block_tree_warps
                Pair v = lane < kWarps ? wparts[b * nloc + j][lane] : pair_identity();
                v = warp_tree_pairs(v);
                if (lane == 0) {  // each word carries the launch's tag: no flag, no fence
                    unsigned long long* w = slots + 2 * (row * a.nb + q + j * G);
                    st_relaxed_gpu_u64(w, tag | __float_as_uint(v.m));
                    st_relaxed_gpu_u64(w + 1, tag | __float_as_uint(v.n));
                }
            }
        }
    };
    auto stats_role = [&]() {  // ------------------------------------------------ statistics warps
        for (int64_t k = warp - kResStatsWarp; k < nrows; k += 2) {
            const int b = ring.rem(k);
            const int64_t row = grp + k * ngroups;
            // every lane loads its leaves' tagged words until all of the row's nb carry this
            // launch's tag: the poll is the load of the values (one round trip once they are in)
            const unsigned long long* rw = slots + 2 * row * a.nb;
            const int l0 = nb > 32 ? 2 * lane : lane, l1 = l0 + 1;
            const bool has0 = l0 < nb, has1 = nb > 32 && l1 < nb;
            Pair p0 = pair_identity(), p1 = pair_identity();
            const unsigned long long t0 = globaltimer_ns();
            unsigned ns = 32;
            for (;;) {
                bool ok = true;
                if (has0) {
                    const unsigned long long m = ld_relaxed_gpu_u64(rw + 2 * l0), n = ld_relaxed_gpu_u64(rw + 2 * l0 + 1);
                    ok = ((m ^ tag) >> 32) == 0 && ((n ^ tag) >> 32) == 0;
                    p0 = Pair{__uint_as_float((unsigned)m), __uint_as_float((unsigned)n)};
                }
                if (has1) {
                    const unsigned long long m = ld_relaxed_gpu_u64(rw + 2 * l1), n = ld_relaxed_gpu_u64(rw + 2 * l1 + 1);
                    ok = ok && ((m ^ tag) >> 32) == 0 && ((n ^ tag) >> 32) == 0;
                    p1 = Pair{__uint_as_float((unsigned)m), __uint_as_float((unsigned)n)};
                }
                if (__all_sync(0xffffffffu, ok)) break;
                if (aborted(err)) return;
                __nanosleep(ns);
                ns = ns < 128 ? ns * 2 : ns;
                if (globaltimer_ns() - t0 > kWaitTimeoutNs) {
                    if (lane == 0) raise_abort(err, 8u);
                    return;
                }
            }
            const Pair root = warp_tree64(nb, [&](int j) { return j == l0 ? p0 : p1; });
            if (lane == 0) {
                s_st[b] = make_float2(__fsub_rn(root.n, 1.0f), __fdiv_rn(0.5f, root.m));
                mbar_arrive(&stats_bar[b]);
            }
        }
    };

    // ------------------------------------------------------------------------ compute warps
    auto pass1_block = [&](int64_t k, int j) -> bool {  // pass 1 of this warp's share of block j of row k
        const int b = ring.rem(k);
        if (!wait_or_abort(&full_bar[b * nloc + j], ph(k), err, 4u)) return false;
        const int valid = (int)min((int64_t)kBlockElems, a.cols - (int64_t)(q + j * G) * kBlockElems);
        BlockVals v;
        load_stage<In>(slot(k, j), v);
        Pair wp = Pair{1.0f, 0.0f};
        const bool cl = (TP_RES_EXP & 8) ? false : warp_pass1<V>(v, valid, &wp);
        if (lane == 0) {
            wparts[b * nloc + j][warp] = wp;
            cbits[b * nloc + j][warp] = cl ? 1 : 0;
            mbar_arrive(&p1_bar[b * nloc + j]);  // release: the warp value before the arrival
        }
        return true;
    };
    auto pass1 = [&](int64_t k) -> bool {
        for (int j = 0; j < nloc; ++j)
            if (!pass1_block(k, j)) return false;
        return true;
    };
    // pass 1 runs `ahead` rows before pass 2: the group exchange of row k (the slowest CTA of the
    // group, the round trip to L2, the row tree) hides behind pass 1 of rows k+1 .. k+ahead,
    // and nbuf - 1 - ahead rows are in flight from HBM
    auto compute_role = [&]() {
        for (int64_t k = 0; k < ahead && k < nrows; ++k)
            if (!pass1(k)) return;
        for (int64_t k = 0; k < nrows; ++k) {
            const int b = ring.rem(k);
            const bool more = k + ahead < nrows;
            const int b1 = ring.rem(k + ahead);
            if (!kResFuse && more && !pass1(k + ahead)) return;
            if (!(TP_RES_EXP & 2) && !wait_or_abort(&stats_bar[b], ph(k), err, 16u)) return;
            const float4 st = (TP_RES_EXP & 2) ? make_float4(3.0f, 0.25f, 0.f, 0.f) : make_float4(s_st[b].x, s_st[b].y, 0.f, 0.f);
            const int64_t row = grp + k * ngroups;
            for (int j = 0; j < nloc; ++j) {  // pass 2 on the staged blocks
                const int64_t e0 = (int64_t)(q + j * G) * kBlockElems;
                const int valid = (int)min((int64_t)kBlockElems, a.cols - e0);
                const bool clamp = cbits[b * nloc + j][warp] != 0;
                if (kResFuse && more) {  // with pass 1 of block j of row k + ahead
                    if (!wait_or_abort(&full_bar[b1 * nloc + j], ph(k + ahead), err, 4u)) return;
                    if (valid == kBlockElems && !clamp) {
                        Pair acc = fused_pass1_pass2<In>(slot(k + ahead, j), slot(k, j), st, a.y + row * a.cols + e0);
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&empty_bar[b * nloc + j]);
                        const bool cl = __any_sync(0xffffffffu, acc_out_of_domain(acc));
                        if (cl) {  // reading G11: the warp's values again, clamped
                            BlockVals v1;
                            load_stage<In>(slot(k + ahead, j), v1);
                            acc = pass1_thread<V, false, true>(v1, valid);
                        }
                        const Pair wp = warp_value(acc);
                        if (lane == 0) {
                            wparts[b1 * nloc + j][warp] = wp;
                            cbits[b1 * nloc + j][warp] = cl ? 1 : 0;
                            mbar_arrive(&p1_bar[b1 * nloc + j]);
                        }
                        continue;
                    }
                    if (!pass1_block(k + ahead, j)) return;
                }
                BlockVals v;
                load_stage<In>(slot(k, j), v);
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty_bar[b * nloc + j]);  // the stage may take the row nbuf ahead
                if (TP_RES_EXP & 4) {  // arithmetic without the stores
                    if (!(TP_RES_EXP & 16)) pass2_thread<false, V>(v, st.x, st.y);
                    float sum = 0.0f;
#pragma unroll
                    for (int i = 0; i < kPerThread; ++i) sum += v.v[i];
                    if (sum == 123.456f) store_block<V>(a.y + row * a.cols + e0, valid, true, v);
                } else
                op_pass2<V>(v, st, clamp, a.y + row * a.cols + e0, valid, true);
            }
        }
    };

    if (warp < kWarps) compute_role();
    else if (warp == kResPostWarp) post_role();
    else if (warp == kResLoadWarp) load_role();
    else stats_role();
    // Every role returns here (also on a watchdog abort): the last CTA out advances the workspace
    // epoch (exit_and_reset), so the next launch's tag differs from every tag written here.
    __syncthreads();
    if (threadIdx.x == 0) exit_and_reset(hdr);
}

// CTAs per row (G) for rows x nb blocks on `sms` SMs, 0 when the schedule does not apply.
// Forced (force_g > 0): any G whose share ceil(nb / G) fits the stages (rows of 4..64 blocks).
// Automatic: one block per CTA and row (G = nb), where the stages hold >= 5 rows, i.e. bf16 rows
// (7 rows of 32 KB): the exchange of a row over G CTAs needs several rows of slack under full HBM
// load (measured, C4 bf16: G = 49 with 7 rows staged 293 us, against the cluster kernel's 318 us
// in the same run; G = 17 / 25 with 2 / 3 rows staged 347-450 us).  fp32 rows stage only 3 blocks
// per SM, too little slack: C4 fp32 424 us against 350 us; they stay on the cluster kernel.  At
// least two rows per group, so that the rows' exchanges overlap.
template <typename In>
int rowres_choose(int64_t rows, int64_t nb, int sms, int force_g) {
    constexpr int B = res_max_local<In>();
    if (nb < 4 || nb > kResMaxNb || rows < 1 || rows >= kResMaxRowsPerGroup) return 0;
    const int gmin = (int)((nb + B - 1) / B);
    if (force_g > 0) return force_g >= gmin && force_g <= nb && force_g <= sms ? force_g : 0;
    if (res_nbuf<In>(1) < 5 || nb > sms || rows < 2 * (sms / nb)) return 0;
    return (int)nb;
}

template <typename In>
cudaError_t launch_rowres(KArgs a, int G, const LaunchOpts& o, cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    const int sms = device_sms(dev);
    if (G < 1 || a.nb > kResMaxNb || (a.nb + G - 1) / G > res_max_local<In>() || !a.ws) return cudaErrorNotSupported;
    int64_t ngroups = (o.grid_ctas > 0 ? o.grid_ctas : sms) / G;
    if (ngroups > a.rows) ngroups = a.rows;
    if (ngroups < 1 || (a.rows + ngroups - 1) / ngroups >= kResMaxRowsPerGroup) return cudaErrorNotSupported;
    const int per = (int)((a.nb + G - 1) / G);
    const int nbuf = res_nbuf<In>(per);
    const size_t dyn = (size_t)nbuf * per * kBlockElems * sizeof(In);
    constexpr int A = kTwoPass;
    auto kern = rowres_kernel<In>;
    static DevCache configured[kMaxDevices];
    if (!configured[dev].load(std::memory_order_acquire)) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kResSmemMax);
        configured[dev].store(1, std::memory_order_release);
    }
    // Two-Pass: pass 1 ahead of pass 2 by `ahead` rows, the other staged rows in flight (measured
    // on C4 bf16, nbuf 7: ahead 3 / 4 / 5 / 6 = 337 / 332 / 335 / 358 us; the exchange's latency
    // under full HBM load needs the slack more than the loads need depth).  Three-Pass: each pass
    // `ahead` rows behind the previous one; Recompute keeps 2 ahead + 1 rows staged, Reload
    // ahead + 1.
    int ahead, lim;
    if (A == kTwoPass) {
        ahead = nbuf >= 5 ? nbuf - 3 : (nbuf > 1 ? nbuf - 1 : 1);
        lim = nbuf - 1;
    } else if (A == kRecompute) {
        ahead = nbuf >= 5 ? 2 : 1;
        lim = (nbuf - 1) / 2;
    } else {
        ahead = nbuf >= 5 ? 3 : 1;
        lim = nbuf - 1;
    }
    if (lim < 1) return cudaErrorNotSupported;
    if (o.lookahead_rows > 0 && o.lookahead_rows <= lim) ahead = (int)o.lookahead_rows;
    if (ahead > lim) ahead = lim;
    last_plan() = Plan{6, A, ngroups * G, G, ahead, nbuf};  // lookahead_rows: rows between passes; hold: rows staged
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(ngroups * G));
    cfg.blockDim = dim3(kResThreads);
    cfg.dynamicSmemBytes = dyn;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a, G, (int)ngroups, nbuf, ahead);
}

template int rowres_choose<float>(int64_t, int64_t, int, int);
template int rowres_choose<uint16_t>(int64_t, int64_t, int, int);
template cudaError_t launch_rowres<float>(KArgs, int, const LaunchOpts&, cudaStream_t);
template cudaError_t launch_rowres<uint16_t>(KArgs, int, const LaunchOpts&, cudaStream_t);

}  // namespace tp
