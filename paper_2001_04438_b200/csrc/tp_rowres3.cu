// Resident-row schedule of the Three-Pass comparators (see tp_rowres.cu for the schedule, the
// roles and the exchange; tp_rowres.cuh for the shared pieces).
#include "tp_rowres.cuh"

namespace tp {

// The Three-Pass comparators on the same schedule (Alg. 1 Recompute PAPER.md:88-104, Alg. 2
// Reload PAPER.md:108-128), so that the Two-Pass is compared on the same footing: every CTA stages
// its share once; compute warps run, per iteration k, the max pass of row k, the Sum-exp pass of
// row k - a (Reload: also y = exp(x - mu)) and the output pass of row k - 2a (Recompute: from
// the staged x; Reload: rescaling y re-read from memory); two exchanges per row (block maxima,
// block sums) through the same tagged slots (word 0: max, word 1: sum), one statistics warp per
// kind.  Block and row reductions are the stream kernel's (bitwise): block max over the 16 warp
// maxima, block sum = perfect tree over the 16 warp sums (one shuffle tree, zero-padded), row
// max / sum = warp_reduce_leaves over the nb block values (one canonical group).
template <typename In, int A>
__global__ void __launch_bounds__(kResThreads, 1) rowres3_kernel(const KArgs a, int G, int ngroups, int nbuf, int ahead) {
    constexpr int V = InTraits<In>::V;
    constexpr int S = kResSlots;
    constexpr bool kRecomp = A == kRecompute;
    extern __shared__ __align__(128) unsigned char dsm[];
    In* stages = reinterpret_cast<In*>(dsm);
    __shared__ __align__(8) uint64_t full_bar[S];
    __shared__ __align__(8) uint64_t pm_bar[S];     // 16 warps done with the max pass of a slot
    __shared__ __align__(8) uint64_t ps_bar[S];     // ... with the Sum-exp pass
    __shared__ __align__(8) uint64_t empty_bar[S];  // ... with the last pass reading the stage
    __shared__ __align__(8) uint64_t mu_bar[S];     // row max of the slot's row formed
    __shared__ __align__(8) uint64_t sg_bar[S];     // row sum formed
    __shared__ float wv[S][kWarps];                 // warp maxima, then warp sums, of a slot
    __shared__ float s_mu[S], s_isg[S];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nb = (int)a.nb;
    const int grp = (int)blockIdx.x / G;
    const int q = (int)blockIdx.x - grp * G;
    const int nloc = (nb - q + G - 1) / G;
    WsHeader* hdr = reinterpret_cast<WsHeader*>(a.ws);
    unsigned* err = &hdr->error;
    if (grp >= ngroups) return;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full_bar[i], 1);
            mbar_init(&pm_bar[i], kWarps);
            mbar_init(&ps_bar[i], kWarps);
            mbar_init(&empty_bar[i], kWarps);
            mbar_init(&mu_bar[i], 1);
            mbar_init(&sg_bar[i], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    pdl_wait_and_release();
    publish_abort_word(a);
    __shared__ unsigned s_epoch;
    if (threadIdx.x == 0) s_epoch = *reinterpret_cast<volatile unsigned*>(&hdr->epoch);
    __syncthreads();
    const unsigned long long tag = (unsigned long long)(s_epoch + 1u) << 32;
    const int64_t nrows = (a.rows - grp + ngroups - 1) / ngroups;
    const ResDiv ring(nbuf);
    auto slot = [&](int64_t k, int j) { return stages + ((size_t)ring.rem(k) * nloc + j) * kBlockElems; };
    auto si = [&](int64_t k, int j) { return ring.rem(k) * nloc + j; };
    auto ph = [&](int64_t k) { return (uint32_t)(ring.quot(k) & 1); };
    auto rowof = [&](int64_t k) { return grp + k * ngroups; };
    unsigned long long* slots = reinterpret_cast<unsigned long long*>(a.ws + a.lay.res_vals);
    const int span = kRecomp ? 2 * ahead : ahead;  // iterations from a row's max pass to its last read of x

    auto load_role = [&]() {
        if (lane != 0) return;
        const In* x = static_cast<const In*>(a.x);
        const uint64_t pol = policy_evict_first();
        auto stage_in = [&](int64_t k, int j) {
            const int64_t e0 = (int64_t)(q + j * G) * kBlockElems;
            const uint32_t bytes = (uint32_t)min((int64_t)kBlockElems, a.cols - e0) * (uint32_t)sizeof(In);
            uint64_t* fb = &full_bar[si(k, j)];
            mbar_arrive_expect_tx(fb, bytes);
            tma_load_1d(slot(k, j), x + rowof(k) * a.cols + e0, bytes, fb, pol);
        };
        for (int64_t k = 0; k < nbuf && k < nrows; ++k)
            for (int j = 0; j < nloc; ++j) stage_in(k, j);
        for (int64_t k = 0; k + nbuf < nrows; ++k)
            for (int j = 0; j < nloc; ++j) {
                if (!wait_or_abort(&empty_bar[si(k, j)], ph(k), err, 2u)) return;
                fence_proxy_async_smem();
                stage_in(k + nbuf, j);
            }
    };
    // block value of slot i (max or sum of the 16 warp values) -> word w of its tagged slot
    auto post = [&](int64_t k, int j, int w) {
        const int i = si(k, j);
        float v;
        if (w == 0) {
            v = warp_max(lane < kWarps ? wv[i][lane] : -__int_as_float(0x7f800000));
        } else {
            v = warp_tree_sum(lane < kWarps ? wv[i][lane] : 0.0f);  // = block_tree_warps_sum
        }
        if (lane == 0) st_relaxed_gpu_u64(slots + 2 * (rowof(k) * a.nb + q + j * G) + w, tag | __float_as_uint(v));
    };
    auto post_role = [&]() {
        for (int64_t k = 0; k < nrows + ahead; ++k) {
            if (k < nrows)
                for (int j = 0; j < nloc; ++j) {
                    if (!wait_or_abort(&pm_bar[si(k, j)], ph(k), err, 32u)) return;
                    post(k, j, 0);
                }
            const int64_t k1 = k - ahead;
            if (k1 >= 0)
                for (int j = 0; j < nloc; ++j) {
                    if (!wait_or_abort(&ps_bar[si(k1, j)], ph(k1), err, 32u)) return;
                    post(k1, j, 1);
                }
        }
    };
    auto stats_role = [&](int w) {  // w = 0: row maxima, 1: row sums
        const int l0 = nb > 32 ? 2 * lane : lane, l1 = l0 + 1;
        const bool has0 = l0 < nb, has1 = nb > 32 && l1 < nb;
        for (int64_t k = 0; k < nrows; ++k) {
            const unsigned long long* rw = slots + 2 * rowof(k) * a.nb + w;
            float f0 = 0.0f, f1 = 0.0f;
            const unsigned long long t0 = globaltimer_ns();
            unsigned ns = 32;
            for (;;) {
                bool ok = true;
                if (has0) {
                    const unsigned long long u = ld_relaxed_gpu_u64(rw + 2 * l0);
                    ok = ((u ^ tag) >> 32) == 0;
                    f0 = __uint_as_float((unsigned)u);
                }
                if (has1) {
                    const unsigned long long u = ld_relaxed_gpu_u64(rw + 2 * l1);
                    ok = ok && ((u ^ tag) >> 32) == 0;
                    f1 = __uint_as_float((unsigned)u);
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
            const int b = ring.rem(k);
            const float2 root = warp_reduce_leaves(w == 0 ? kRedMax : kRedSum, nb,
                                                   [&](int64_t j) { return make_float2(j == l0 ? f0 : f1, 0.0f); });
            if (w == 0) {
                if (lane == 0) {
                    s_mu[b] = root.x;
                    mbar_arrive(&mu_bar[b]);
                }
            } else {
                if (!wait_or_abort(&mu_bar[b], ph(k), err, 16u)) return;  // s_mu of the row is in
                const float4 st = row_stats_of<A>(1, root, s_mu[b]);
                if (lane == 0) {
                    s_isg[b] = st.y;
                    mbar_arrive(&sg_bar[b]);
                }
            }
        }
    };
    auto compute_role = [&]() {
        for (int64_t k = 0; k < nrows + span; ++k) {
            if (k < nrows) {  // max pass of row k
                for (int j = 0; j < nloc; ++j) {
                    const int i = si(k, j);
                    if (!wait_or_abort(&full_bar[i], ph(k), err, 4u)) return;
                    const int valid = (int)min((int64_t)kBlockElems, a.cols - (int64_t)(q + j * G) * kBlockElems);
                    BlockVals v;
                    load_stage<In>(slot(k, j), v);
                    const float m = warp_max(valid == kBlockElems ? max_thread<V, true>(v, valid)
                                                                  : max_thread<V, false>(v, valid));
                    if (lane == 0) {
                        wv[i][warp] = m;
                        mbar_arrive(&pm_bar[i]);
                    }
                }
            }
            const int64_t k1 = k - ahead;
            if (k1 >= 0 && k1 < nrows) {  // Sum-exp pass of row k1
                const int b = ring.rem(k1);
                if (!wait_or_abort(&mu_bar[b], ph(k1), err, 16u)) return;
                const float mu = s_mu[b];
                for (int j = 0; j < nloc; ++j) {
                    const int i = si(k1, j);
                    const int64_t e0 = (int64_t)(q + j * G) * kBlockElems;
                    const int valid = (int)min((int64_t)kBlockElems, a.cols - e0);
                    BlockVals v;
                    load_stage<In>(slot(k1, j), v);
                    if (!kRecomp) {  // Reload: the stage is free after this pass
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&empty_bar[i]);
                    }
                    float sm = valid == kBlockElems ? exp_sum_thread<V, true>(v, valid, mu)
                                                    : exp_sum_thread<V, false>(v, valid, mu);
                    if (!kRecomp) store_block<V>(a.y + rowof(k1) * a.cols + e0, valid, true, v);  // Y = Exp(X - mu)
                    sm = warp_tree_sum(sm);
                    if (lane == 0) {
                        wv[i][warp] = sm;
                        mbar_arrive(&ps_bar[i]);
                    }
                }
            }
            const int64_t k2 = k - span;
            if (k2 >= 0 && k2 < nrows) {  // output pass of row k2
                const int b = ring.rem(k2);
                if (!wait_or_abort(&sg_bar[b], ph(k2), err, 16u)) return;
                const float4 st = make_float4(s_mu[b], s_isg[b], 0.f, 0.f);
                for (int j = 0; j < nloc; ++j) {
                    const int64_t e0 = (int64_t)(q + j * G) * kBlockElems;
                    const int valid = (int)min((int64_t)kBlockElems, a.cols - e0);
                    float* yb = a.y + rowof(k2) * a.cols + e0;
                    if (kRecomp) {
                        BlockVals v;
                        load_stage<In>(slot(k2, j), v);
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&empty_bar[si(k2, j)]);
                        op_out_recompute<V>(v, st, yb, valid, true);
                    } else {
                        op_out_reload(st, yb, valid, true);
                    }
                }
            }
        }
    };

    if (warp < kWarps) compute_role();
    else if (warp == kResPostWarp) post_role();
    else if (warp == kResLoadWarp) load_role();
    else stats_role(warp - kResStatsWarp);
    __syncthreads();
    if (threadIdx.x == 0) exit_and_reset(hdr);
}

template <typename In, int A>
cudaError_t launch_rowres3(KArgs a, int G, const LaunchOpts& o, cudaStream_t s) {
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
    auto kern = rowres3_kernel<In, A>;
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

template cudaError_t launch_rowres3<float, kRecompute>(KArgs, int, const LaunchOpts&, cudaStream_t);
template cudaError_t launch_rowres3<uint16_t, kRecompute>(KArgs, int, const LaunchOpts&, cudaStream_t);
template cudaError_t launch_rowres3<float, kReload>(KArgs, int, const LaunchOpts&, cudaStream_t);
template cudaError_t launch_rowres3<uint16_t, kReload>(KArgs, int, const LaunchOpts&, cudaStream_t);

}  // namespace tp
