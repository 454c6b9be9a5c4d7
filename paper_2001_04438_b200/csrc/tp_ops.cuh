// Per-item operations shared by the warp-specialised TMA kernel (tp_stream.cu) and the general
// kernel (tp_kernels.cu), so both compute bit-identical results.
//
// Compute side (every compute warp, on its 32 x 32 values of the block):
//   op_pass1        Alg. 3 pass 1: warp pair + clamp decision -> part[w]
//   op_pass2        Alg. 3 pass 2 -> y
//   op_fused_tail   rows of one block: block pair from part[], lambda, pass 2 -> y
//   op_max / op_expsum / op_out_*   Three-Pass passes
// Retire side (one warp): the block value from part[], publication and row finishing.
#pragma once
#include "tp_sched.cuh"

namespace tp {

struct Part {
    Pair v[kWarps];           // per-warp pair (Two-Pass) or value in .m (max / sum)
    unsigned char cb[kWarps]; // per-warp clamp decision of pass 1
};

template <int V>
__device__ __forceinline__ void op_pass1(const BlockVals& r, int valid, Part& part) {
    Pair wp;
    const bool cl = warp_pass1<V>(r, valid, &wp);
    if ((threadIdx.x & 31) == 0) {
        part.v[threadIdx.x >> 5] = wp;
        part.cb[threadIdx.x >> 5] = cl ? 1 : 0;
    }
}

template <int V>
__device__ __forceinline__ void op_pass2(BlockVals& r, float4 st, bool clamp, float* yb, int valid, bool vec,
                                         int tid = (int)threadIdx.x) {
    if (vec && valid == kBlockElems) {
        if (clamp) pass2_store_full<V, true>(r, st.x, st.y, yb, tid);
        else pass2_store_full<V, false>(r, st.x, st.y, yb, tid);
        return;
    }
    if (clamp) pass2_thread<true, V>(r, st.x, st.y, valid, tid);
    else pass2_thread<false, V>(r, st.x, st.y, valid, tid);
    store_block<V>(yb, valid, vec, r, tid);
}

// After every compute warp has run op_pass1 and a barrier among them: the row pair is the
// block pair (one block per row), lambda' and pass 2 on the same staged values.
template <int V>
__device__ __forceinline__ void op_fused_tail(BlockVals& r, const Part& part, float* yb, int valid, bool vec) {
    const Pair root = block_tree_warps(part.v);
    const float4 st = make_float4(__fsub_rn(root.n, 1.0f), __fdiv_rn(0.5f, root.m), 0.0f, 0.0f);
    op_pass2<V>(r, st, part.cb[threadIdx.x >> 5] != 0, yb, valid, vec);
}

template <int V>
__device__ __forceinline__ void op_max(const BlockVals& r, int valid, Part& part) {
    const float m = warp_max(valid == kBlockElems ? max_thread<V, true>(r, valid) : max_thread<V, false>(r, valid));
    if ((threadIdx.x & 31) == 0) part.v[threadIdx.x >> 5] = Pair{m, 0.0f};
}

template <int V, bool RELOAD>
__device__ __forceinline__ void op_expsum(BlockVals& r, int valid, float mu, Part& part, float* yb, bool vec) {
    float s = valid == kBlockElems ? exp_sum_thread<V, true>(r, valid, mu) : exp_sum_thread<V, false>(r, valid, mu);
    if (RELOAD) store_block<V>(yb, valid, vec, r);  // Y_i <- Exp(X_i - mu)
    s = warp_tree_sum(s);
    if ((threadIdx.x & 31) == 0) part.v[threadIdx.x >> 5] = Pair{s, 0.0f};
}

template <int V>
__device__ __forceinline__ void op_out_recompute(BlockVals& r, float4 st, float* yb, int valid, bool vec) {
    if (valid == kBlockElems) exp_sum_thread<V, true>(r, valid, st.x);
    else exp_sum_thread<V, false>(r, valid, st.x);
    scale_thread(r, st.y);  // Y_i <- lambda * Exp(X_i - mu)
    store_block<V>(yb, valid, vec, r);
}

__device__ __forceinline__ void op_out_reload(float4 st, float* yb, int valid, bool yvec) {
    BlockVals r;
    load_global_y(yb, valid, yvec, r);
    scale_thread(r, st.y);  // Y_i <- lambda * Y_i
    store_block<4>(yb, valid, yvec, r);
}

// Does finishing this item publish a block value?  (Two-Pass pass 1; Three-Pass passes 1-2)
template <int A>
__device__ __forceinline__ bool item_retires(const Item& it) {
    return ((A == kTwoPass || A == kPartial) && it.phase == 0) || ((A == kRecompute || A == kReload) && it.phase < 2);
}

// The block's value from its warp values (one thread): the pair tree (plus the block's clamp
// mask, stored for pass 2 and flagged on the row), the max, or the sum tree.
template <int A>
__device__ __forceinline__ float2 block_value(const KArgs& a, const Item& it, const Part& part) {
    const int kind = red_kind<A>(it.phase);
    if (kind == kRedPair) {
        const Pair bp = block_tree_warps(part.v);
        unsigned mask = 0;
        for (int w = 0; w < kWarps; ++w) mask |= (unsigned)part.cb[w] << w;
        // every block's mask is stored (0 included), so a row with some clamped block never
        // reads another block's stale mask from an earlier launch
        reinterpret_cast<unsigned*>(a.ws + a.lay.block_clamp)[it.row * a.nb + it.blk] = mask;
        if (mask) atomicOr(reinterpret_cast<unsigned*>(a.ws + a.lay.row_clamp) + it.row, 1u);
        return make_float2(bp.m, bp.n);
    }
    if (kind == kRedMax) {
        float m = part.v[0].m;
        for (int w = 1; w < kWarps; ++w) m = fmaxf(m, part.v[w].m);
        return make_float2(m, 0.0f);
    }
    float s[kWarps];
    for (int w = 0; w < kWarps; ++w) s[w] = part.v[w].m;
    return make_float2(block_tree_warps_sum(s), 0.0f);
}

// Fused one-sided exchange, push side (one thread, when a row's pass-1 pair is final): store
// the pair into slot `rank` of every mailbox (P2P stores over NVLink), make it visible
// system-wide, count the row; the thread that completes the launch's last row releases the
// exchange epoch into flag `rank` of every mailbox (after its own system fence, so every row's
// stores, each fenced before its count, precede the flag).  The count returns to 0 for the next
// launch.
__device__ __forceinline__ void push_row_pair(const KArgs& a, int64_t row, float2 root) {
    const size_t off = mailbox_pairs_offset(a.world, a.rows, a.xepoch);
    for (int p = 0; p < a.world; ++p)
        reinterpret_cast<float2*>(a.peers[p] + off)[(int64_t)a.rank * a.rows + row] = root;
    __threadfence_system();
    WsHeader* hdr = reinterpret_cast<WsHeader*>(a.ws);
    if (atomicAdd(&hdr->rows_done, 1u) == (unsigned)(a.rows - 1)) {
        hdr->rows_done = 0u;
        __threadfence_system();
        for (int p = 0; p < a.world; ++p)
            st_release_sys(reinterpret_cast<unsigned*>(a.peers[p] + mailbox_flag_offset(a.xepoch, a.rank)), a.xepoch);
    }
}

// Fused one-sided exchange, wait side (one thread per CTA, before its first kFinish item):
// acquire the world flags of the local mailbox for this epoch.  A peer missing for wait_ns sets
// its bit in the mailbox error word and watchdog bit 0 (the launch then runs on whatever pairs
// are there, as after the separate wait kernel; the host reads the flags).
__device__ __forceinline__ void finish_wait(const KArgs& a) {
    const unsigned long long t0 = globaltimer_ns();
    for (int p = 0; p < a.world; ++p) {
        const unsigned* flag = reinterpret_cast<const unsigned*>(a.mailbox + mailbox_flag_offset(a.xepoch, p));
        while (ld_acquire_sys(flag) != a.xepoch) {
            if (globaltimer_ns() - t0 > a.wait_ns) {
                atomicOr(reinterpret_cast<unsigned*>(const_cast<char*>(a.mailbox) + kMailboxErrorWord), 1u << (p & 31));
                raise_abort(&reinterpret_cast<WsHeader*>(a.ws)->error, 1u);
                break;
            }
            __nanosleep(128);
        }
    }
}

// Publish a batch of block values (one whole warp; each lane with `mine` holds one item's
// value): every lane stores its value, ONE fence covers the batch, every lane takes its group
// ticket; then each group completed by the batch is reduced by the warp (canonical tree), and
// a row completed by that group is reduced and released.
template <int A>
__device__ void retire_batch(const KArgs& a, bool mine, const Item& it, float2 val, float mu, unsigned want) {
    const int lane = threadIdx.x & 31;
    float2* block_vals = reinterpret_cast<float2*>(a.ws + a.lay.block_vals);
    float2* group_vals = reinterpret_cast<float2*>(a.ws + a.lay.group_vals);
    unsigned* gt = reinterpret_cast<unsigned*>(a.ws + a.lay.group_tickets);
    unsigned* rt = reinterpret_cast<unsigned*>(a.ws + a.lay.row_tickets);
    unsigned* row_clamp = reinterpret_cast<unsigned*>(a.ws + a.lay.row_clamp);
    const int64_t g = it.blk / kGroupBlocks;
    bool last = false;
    if (mine) {
        block_vals[it.row * a.nb + it.blk] = val;
        const int64_t gsize = min((int64_t)kGroupBlocks, a.nb - g * kGroupBlocks);
        // release: this lane's block value before its ticket; acquire: the group's last ticket
        // sees every other block value of the group (their tickets released them)
        last = atom_add_acq_rel_gpu(&gt[it.row * a.ng + g], 1u) == (unsigned)(gsize - 1);
    }
    unsigned fin = __ballot_sync(0xffffffffu, last);
    if (!fin) return;
    __syncwarp();  // the acquiring lanes' view passes to the whole warp (warp barrier orders memory)
    while (fin) {
        const int l = __ffs(fin) - 1;
        fin &= fin - 1;
        const int phase = __shfl_sync(0xffffffffu, it.phase, l);
        const int64_t row = __shfl_sync(0xffffffffu, it.row, l);
        const int64_t gg = __shfl_sync(0xffffffffu, g, l);
        const float mu_l = __shfl_sync(0xffffffffu, mu, l);
        const int kind = red_kind<A>(phase);
        const int64_t gsize = min((int64_t)kGroupBlocks, a.nb - gg * kGroupBlocks);
        const float2* gv = block_vals + row * a.nb + gg * kGroupBlocks;
        const float2 gres = warp_reduce_leaves(kind, gsize, [&](int64_t j) { return __ldcg(gv + j); });
        unsigned rlast = 0;
        if (lane == 0) {
            gt[row * a.ng + gg] = 0u;  // ticket reset for the next phase / launch
            group_vals[row * a.ng + gg] = gres;
            rlast = atom_add_acq_rel_gpu(&rt[row], 1u) == (unsigned)(a.ng - 1);
        }
        if (!__shfl_sync(0xffffffffu, rlast, 0)) continue;
        __syncwarp();
#ifdef TP_PH_PROF  // development timeline (tools/prof_phase.py): the row tree's start and end
        if (a.prof && lane == 0) a.prof[16 + 5 * 200] = globaltimer_ns();
#endif
        const float2* rv = group_vals + row * a.ng;
        const float2 root = warp_reduce_leaves(kind, a.ng, [&](int64_t j) { return __ldcg(rv + j); });
#ifdef TP_PH_PROF
        if (a.prof && lane == 0) a.prof[16 + 5 * 200 + 1] = globaltimer_ns();
#endif
        if (lane == 0) {
            rt[row] = 0u;
            float clamped = 0.0f;  // did any block of the row take the clamped path?
            if (A == kTwoPass || A == kPartial) {
                clamped = __ldcg(&row_clamp[row]) ? 1.0f : 0.0f;
                row_clamp[row] = 0u;
            }
            if (A == kPartial) {
                // the chunk's clamp flag stays in the workspace for the finish launch on it
                reinterpret_cast<float4*>(a.ws + a.lay.row_stats)[row * 2] = make_float4(root.x, root.y, clamped, 0.f);
                if (a.pair_out) a.pair_out[row] = root;
                if (a.peers) push_row_pair(a, row, root);
            } else {
                if ((A == kRecompute || A == kReload) && a.shard_out) a.shard_out[row] = root.x;  // sharded
                float4 st = row_stats_of<A>(phase, root, mu_l);
                if (A == kTwoPass) st.z = clamped;
                reinterpret_cast<float4*>(a.ws + a.lay.row_stats)[row * 2 + phase] = st;
                st_release_gpu(reinterpret_cast<unsigned*>(a.ws + a.lay.row_ready) + row * 2 + phase, want);
            }
        }
    }
}

// Retire a phase's block (one whole warp, value from lane 0's view of the warp parts).
template <int A>
__device__ __forceinline__ void retire_block(const KArgs& a, const Item& it, const Part& part, unsigned want,
                                             float mu) {
    const int lane = threadIdx.x & 31;
    float2 val = make_float2(0.0f, 0.0f);
    if (lane == 0) val = block_value<A>(a, it, part);
    retire_batch<A>(a, lane == 0, it, val, mu, want);
}

// Statistics a later-phase item needs: (stats, per-warp clamp mask).  Called by one thread
// after the row's previous phase has been released.  The per-block mask is read only when
// some block of the row took the clamped path (stats.z, rare).
template <int A>
__device__ __forceinline__ void item_stats(const KArgs& a, const Item& it, float4* st, unsigned* mask) {
    const float4* row_stats = reinterpret_cast<const float4*>(a.ws + a.lay.row_stats);
    *st = __ldcg(row_stats + it.row * 2 + (it.phase - 1));
    *mask = 0;
    if (A == kTwoPass && st->z != 0.0f)
        *mask = __ldcg(reinterpret_cast<const unsigned*>(a.ws + a.lay.block_clamp) + it.row * a.nb + it.blk);
}

// kFinish: merge the world partials of a row with the canonical tree over rank index.  .z: did
// the partial launch on this workspace clamp any block of the row's chunk (reading G11; the
// per-block masks are then in the workspace)?
__device__ __forceinline__ float4 finish_stats(const KArgs& a, int64_t row) {
    const Pair root = seq_tree_pairs((int)next_pow2(a.world), [&](int i) {
        if (i >= a.world) return pair_identity();
        const float2 v = a.pairs_in[(int64_t)i * a.rows + row];
        return Pair{v.x, v.y};
    });
    const float clamped = __ldcg(reinterpret_cast<const float4*>(a.ws + a.lay.row_stats) + row * 2).z;
    return make_float4(__fsub_rn(root.n, 1.0f), __fdiv_rn(0.5f, root.m), clamped, 0.0f);
}

// kFinish: the per-warp clamp decisions the partial launch took for this block (0 when no block
// of the row's chunk was clamped).
__device__ __forceinline__ unsigned finish_mask(const KArgs& a, const float4& st, int64_t row, int64_t blk) {
    return st.z != 0.0f ? __ldcg(reinterpret_cast<const unsigned*>(a.ws + a.lay.block_clamp) + row * a.nb + blk) : 0u;
}

// Sharded Three-Pass: the statistics a phase needs from the world's gathered partials.  mu = the
// max over ranks (exact); sigma = the canonical tree over rank index of the ranks' sums (reading
// G8: with power-of-two worlds and chunks the ranks' sums are subtrees of the one-GPU tree, so
// the result is bitwise that of one GPU).  dep_phase 0: (mu); 1: (mu, 1 / sigma, sigma).
template <int A>
__device__ __forceinline__ float4 shard_stats(const KArgs& a, int64_t row, int dep_phase) {
    float mu = -__int_as_float(0x7f800000);
    for (int w = 0; w < a.world; ++w) mu = fmaxf(mu, a.shard_mu[(int64_t)w * a.rows + row]);
    if (dep_phase == 0) return make_float4(mu, 0.0f, 0.0f, 0.0f);
    const float sigma = seq_tree_sum((int)next_pow2(a.world), [&](int i) {
        return i < a.world ? a.shard_sigma[(int64_t)i * a.rows + row] : 0.0f;
    });
    return row_stats_of<A>(1, make_float2(sigma, 0.0f), mu);
}

template <int A>
__device__ __forceinline__ bool item_needs_stats(const Item& it) {
    return (AlgoTraits<A>::P > 1 && it.phase > 0) || A == kFinish;
}

// warp_reduce_leaves(kRedPair, n, leaf) for n <= 64, registers only, result in every lane:
// lane l reduces leaves [l c, l c + c) (c = 2 when next_pow2(n) = 64, else 1), then the warp tree.
template <typename LeafFn>
__device__ __forceinline__ Pair warp_tree64(int n, LeafFn leaf) {
    const int lane = threadIdx.x & 31;
    Pair v = pair_identity();
    if (n > 32) {
        const int b = 2 * lane;
        if (b < n) v = pair_merge(leaf(b), b + 1 < n ? leaf(b + 1) : pair_identity());
    } else if (lane < n) {
        v = leaf(lane);
    }
    v = warp_tree_pairs(v);
    return Pair{__shfl_sync(0xffffffffu, v.m, 0), __shfl_sync(0xffffffffu, v.n, 0)};
}

// host side (tp_kernels.cu / tp_stream.cu)
int device_sms(int dev);
int64_t lookahead_rows(const KArgs& a, int64_t grid, int items_per_cta, const LaunchOpts& o);
template <typename In, int A>
cudaError_t launch_stream(KArgs a, const LaunchOpts& o, cudaStream_t s);
bool small_applies(int64_t rows, int64_t nb, int vec);
template <typename In, int A>
cudaError_t launch_small(KArgs a, const LaunchOpts& o, cudaStream_t s);
template <typename In>
int rowcl_choose(int64_t rows, int64_t nb, int force_cl, bool vs_stream, int64_t* tail_rows, int* tail_ctas,
                 int* tail_cl);
template <typename In>
cudaError_t launch_rowcl(KArgs a, int CL, const LaunchOpts& o, cudaStream_t s);
template <typename In, int A>
cudaError_t launch_rowcl3(KArgs a, int CL, const LaunchOpts& o, cudaStream_t s);
bool rowph_applies(int A, int64_t rows, int64_t nb, int sms);
template <typename In, int A>
cudaError_t launch_rowph(KArgs a, const LaunchOpts& o, cudaStream_t s);
template <typename In>
int rowres_choose(int64_t rows, int64_t nb, int sms, int force_g);
template <typename In>
cudaError_t launch_rowres(KArgs a, int G, const LaunchOpts& o, cudaStream_t s);
template <typename In, int A>
cudaError_t launch_rowres3(KArgs a, int G, const LaunchOpts& o, cudaStream_t s);

}  // namespace tp
