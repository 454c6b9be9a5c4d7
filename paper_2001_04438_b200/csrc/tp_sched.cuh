// Work items, workspace layout and the cross-CTA reduction protocol shared by the kernels.
//
// A launch processes rows x nb blocks per phase (nb = ceil(cols / kBlockElems)).  Items are
// handed out by an in-order atomic queue (WsHeader::counter).  For multi-phase algorithms the
// queue interleaves rows: schedule slot s holds phase p of row s - p*L, oldest phase first, so
// a row's later phase is reached about L rows after its first (reading of the paper's pass
// structure onto a persistent grid).
//
// Reduction protocol (reading G8, canonical tree): a finished block publishes its value, then
// increments its group's ticket; the block that completes a group of kGroupBlocks reduces it
// (perfect tree over the padded group), the group that completes the row reduces the group
// values (perfect tree over the padded group count).  Equal to the perfect tree over the row's
// nb block values padded to a power of two, whatever the grid, timing or arrival order.
#pragma once
#include "tp_block.cuh"
#include "tp_internal.h"

namespace tp {

__host__ __device__ inline size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

// Control region first (header, tickets, row flags: zero when a launch starts; the kernels
// leave it that way except for the epoch-tagged ready flags), then the data region.
__host__ __device__ inline WsLayout ws_layout(int64_t rows, int64_t cols) {
    WsLayout L{};
    const int64_t nb = (cols + kBlockElems - 1) / kBlockElems;
    const int64_t ng = (nb + kGroupBlocks - 1) / kGroupBlocks;
    size_t off = align256(sizeof(WsHeader));
    L.group_tickets = off; off = align256(off + sizeof(unsigned) * rows * ng);
    L.row_tickets = off;   off = align256(off + sizeof(unsigned) * rows);
    L.row_ready = off;     off = align256(off + sizeof(unsigned) * rows * 2);
    L.row_clamp = off;     off = align256(off + sizeof(unsigned) * rows);
    // in the control region: zero-filled with the header on a shape change, so that no tag of a
    // previous shape's launch can equal a tag of this shape's epochs (tp_rowres.cu)
    L.res_vals = off;      off = align256(off + 16 * rows * (nb <= kGroupBlocks ? nb : 0));
    L.ctrl_bytes = off;
    L.row_stats = off;     off = align256(off + sizeof(float4) * rows * 2);
    L.block_vals = off;    off = align256(off + sizeof(float2) * rows * nb);
    L.block_clamp = off;   off = align256(off + sizeof(unsigned) * rows * nb);
    L.group_vals = off;    off = align256(off + sizeof(float2) * rows * ng);
    L.bytes = off;
    return L;
}

enum Algo : int { kTwoPass = 0, kPartial = 1, kRecompute = 2, kReload = 3, kFused = 4, kFinish = 5 };

template <int A> struct AlgoTraits { static constexpr int P = 1; };
template <> struct AlgoTraits<kTwoPass> { static constexpr int P = 2; };
template <> struct AlgoTraits<kRecompute> { static constexpr int P = 3; };
template <> struct AlgoTraits<kReload> { static constexpr int P = 3; };

struct KArgs {
    const void* x;
    float* y;
    int64_t rows, cols, nb, ng;
    int64_t L;              // lookahead in rows
    int64_t total_items;    // rows * nb * phases
    char* ws;
    WsLayout lay;
    float2* pair_out;        // kPartial: one (m, n) per row
    const float2* pairs_in;  // kFinish: world x rows pairs, rank-major
    int world;
    int vec;                 // 16-byte aligned rows
    int l2_hints;            // TMA loads carry evict_last / evict_first L2 policies
    int hold;                // stream kernel: blocks stay staged between pass 1 and pass 2
    int phase_only;          // measurement (tp_phase_only): 1 + the one phase this launch runs, else 0
    // fused one-sided NVLink exchange (tp_peer.cu mailbox layout):
    char* const* peers;      // kPartial: world mailboxes (device array) the row pairs are pushed to, or null
    int rank;                // kPartial: this rank's slot in every mailbox
    unsigned xepoch;         // exchange epoch released into flag `rank` (kPartial) / awaited (kFinish)
    const char* mailbox;     // kFinish: the local mailbox whose flags are awaited in-kernel, or null
    unsigned long long wait_ns;  // kFinish: give up (error bits) after this long
    unsigned long long* prof;  // development: per-role cycle counters (tp_set_profile_buffer), or null
    unsigned* abort_host;      // host-mapped abort word of the device (WsHeader::abort_host)
    // sharded Three-Pass (softmax3_*_partial / finish, phase_only launches): the world's
    // gathered per-row maxima and sums (world x rows, rank-major), and this launch's per-row
    // result (max or sum of the local chunk), or null
    const float* shard_mu;
    const float* shard_sigma;
    float* shard_out;
};

// Record a watchdog abort: the launch's error bit (every role polls it and leaves) and the
// device's host-mapped word, so the next C-ABI call returns TP_EWATCHDOG (a plain system-scope
// store of 1: idempotent, no host-memory atomics needed).  err is &WsHeader::error.
__device__ __forceinline__ void raise_abort(unsigned* err, unsigned bit) {
    atomicOr(err, bit);
    const WsHeader* h = reinterpret_cast<const WsHeader*>(reinterpret_cast<const char*>(err) - offsetof(WsHeader, error));
    unsigned* host = *reinterpret_cast<unsigned* const volatile*>(&h->abort_host);
    if (host) {
        *reinterpret_cast<volatile unsigned*>(host) = 1u;
        __threadfence_system();
    }
}

// First thread of a launch: publish the abort word in the workspace header it uses.
__device__ __forceinline__ void publish_abort_word(const KArgs& a) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.ws)
        reinterpret_cast<WsHeader*>(a.ws)->abort_host = a.abort_host;
}

// number of (phase, row) units in schedule slots < s.  Item arithmetic is 32-bit: a launch
// has far fewer than 2^32 items (2^32 blocks would be 2^46 elements).
__device__ __forceinline__ uint32_t units_before(uint32_t s, uint32_t R, uint32_t L, int P) {
    uint32_t c = 0;
    for (int p = 0; p < P; ++p) {
        const uint32_t off = (uint32_t)p * L;
        const uint32_t v = s > off ? s - off : 0u;
        c += v > R ? R : v;
    }
    return c;
}

struct Item {
    int phase;
    int64_t row, blk;
};

template <int A>
__device__ __forceinline__ Item decode_item(int64_t item64, int64_t R64, int64_t nb64, int64_t L64) {
    constexpr int P = AlgoTraits<A>::P;
    const uint32_t item = (uint32_t)item64, R = (uint32_t)R64, nb = (uint32_t)nb64, L = (uint32_t)L64;
    Item it;
    const uint32_t unit = item / nb;
    const uint32_t bi = item - unit * nb;
    if (P == 1) {
        it.phase = 0;
        it.row = unit;
        it.blk = (A == kFinish) ? nb - 1 - bi : bi;  // pass 2 walks backwards (L2 tail first)
        return it;
    }
    uint32_t lo = 0, hi = R + (uint32_t)(P - 1) * L;  // slot s: units_before(s) <= unit < units_before(s+1)
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (units_before(mid, R, L, P) <= unit) lo = mid; else hi = mid;
    }
    const uint32_t s = lo;
    const uint32_t pmax = (uint32_t)(P - 1);
    const int p_hi = (int)min(s / L, pmax);
    const uint32_t idx = unit - units_before(s, R, L, P);
    it.phase = p_hi - (int)idx;  // within a slot: oldest row (highest phase) first
    it.row = s - (uint32_t)it.phase * L;
    it.blk = it.phase > 0 ? nb - 1 - bi : bi;
    return it;
}

// What a phase reduces: pairs (Two-Pass pass 1), a max (Three-Pass pass 1), a sum (pass 2).
enum RedKind : int { kRedPair = 0, kRedMax = 1, kRedSum = 2 };

template <int A>
__device__ __forceinline__ int red_kind(int phase) {
    if (A == kRecompute || A == kReload) return phase == 0 ? kRedMax : kRedSum;
    return kRedPair;
}

// Canonical warp-level reduction of n leaves (perfect tree over the padded power of two):
// lane l reduces leaves [l*c, (l+1)*c) in order, then the 32 lane results are tree-reduced.
// With c >= kLeafChunk a lane loads its leaves a chunk at a time with independent loads (a row
// of 2048 groups would otherwise wait on 64 dependent L2 round trips per lane: ~40 us at the end
// of C5's pass 1); each chunk's perfect subtree, then the chunks' perfect tree, is the perfect
// tree over the c leaves.
constexpr int kLeafChunk = 8;
template <typename LeafFn>
__device__ __forceinline__ float2 warp_reduce_leaves(int kind, int64_t n, LeafFn leaf) {
    const int lane = threadIdx.x & 31;
    const int64_t P = next_pow2(n);
    const int64_t c = P > 32 ? P / 32 : 1;
    const int64_t base = (int64_t)lane * c;
    constexpr int K = kLeafChunk;
    const float ninf = -__int_as_float(0x7f800000);
    // chunk j of this lane's leaves (c >= K), positions past n hold `pad`
    auto load_chunk = [&](int64_t j, float2 pad, float2 (&f)[K]) {
#pragma unroll
        for (int i = 0; i < K; ++i) {
            const int64_t q = base + j * K + i;
            f[i] = q < n ? leaf(q) : pad;
        }
    };
    if (kind == kRedMax) {
        float m = ninf;
        if (c >= K) {
            for (int64_t j = 0; j < c / K && base + j * K < n; ++j) {
                float2 f[K];
                load_chunk(j, make_float2(ninf, 0.0f), f);
#pragma unroll
                for (int i = 0; i < K; ++i) m = fmaxf(m, f[i].x);
            }
        } else {
            for (int64_t j = base; j < base + c && j < n; ++j) m = fmaxf(m, leaf(j).x);
        }
        return make_float2(warp_max(m), 0.0f);
    }
    if (kind == kRedSum) {
        float v = 0.0f;
        if (base < n) {
            if (c >= K) {
                v = seq_tree_sum((int)(c / K), [&](int j) {
                    float2 f[K];
                    load_chunk(j, make_float2(0.0f, 0.0f), f);
#pragma unroll
                    for (int o = 1; o < K; o <<= 1)
#pragma unroll
                        for (int i = 0; i + o < K; i += 2 * o) f[i].x = __fadd_rn(f[i].x, f[i + o].x);
                    return f[0].x;
                });
            } else {
                v = seq_tree_sum((int)c, [&](int i) { return base + i < n ? leaf(base + i).x : 0.0f; });
            }
        }
        return make_float2(warp_tree_sum(v), 0.0f);
    }
    Pair v = pair_identity();
    if (base < n) {
        if (c >= K) {
            v = seq_tree_pairs((int)(c / K), [&](int j) {
                float2 f[K];
                load_chunk(j, make_float2(0.0f, ninf), f);  // (0, -inf): the identity
                return tree_pairs_n<K>([&](int i) { return Pair{f[i].x, f[i].y}; });
            });
        } else {
            v = seq_tree_pairs((int)c, [&](int i) {
                if (base + i >= n) return pair_identity();
                const float2 f = leaf(base + i);
                return Pair{f.x, f.y};
            });
        }
    }
    v = warp_tree_pairs(v);
    return make_float2(v.m, v.n);
}

// Executed by one whole warp.  Publishes block `blk` of `row` (value in lane 0) and, if it
// completes its group and then its row, reduces them.  Returns true (warp-uniform) when this
// warp finished the row; the row value is then in lane 0 of *root.
template <int A>
__device__ bool publish_warp(const KArgs& a, int phase, int64_t row, int64_t blk, float2 val, float2* root) {
    const int lane = threadIdx.x & 31;
    float2* block_vals = reinterpret_cast<float2*>(a.ws + a.lay.block_vals);
    float2* group_vals = reinterpret_cast<float2*>(a.ws + a.lay.group_vals);
    unsigned* gt = reinterpret_cast<unsigned*>(a.ws + a.lay.group_tickets);
    unsigned* rt = reinterpret_cast<unsigned*>(a.ws + a.lay.row_tickets);
    const int kind = red_kind<A>(phase);
    const int64_t g = blk / kGroupBlocks;
    const int64_t gsize = min((int64_t)kGroupBlocks, a.nb - g * kGroupBlocks);
    unsigned last = 0;
    if (lane == 0) {
        block_vals[row * a.nb + blk] = val;
        __threadfence();
        last = (atomicAdd(&gt[row * a.ng + g], 1u) == (unsigned)(gsize - 1));
    }
    if (!__shfl_sync(0xffffffffu, last, 0)) return false;
    __threadfence();
    const float2* gv = block_vals + row * a.nb + g * kGroupBlocks;
    const float2 gres = warp_reduce_leaves(kind, gsize, [&](int64_t j) { return __ldcg(gv + j); });
    last = 0;
    if (lane == 0) {
        gt[row * a.ng + g] = 0u;  // ticket reset for the next phase / launch
        group_vals[row * a.ng + g] = gres;
        __threadfence();
        last = (atomicAdd(&rt[row], 1u) == (unsigned)(a.ng - 1));
    }
    if (!__shfl_sync(0xffffffffu, last, 0)) return false;
    __threadfence();
    const float2* rv = group_vals + row * a.ng;
    *root = warp_reduce_leaves(kind, a.ng, [&](int64_t j) { return __ldcg(rv + j); });
    if (lane == 0) rt[row] = 0u;
    return true;
}

// Row statistics published by a finished phase.  Two-Pass: (n_sum - 1, lambda' = 0.5 / m_sum)
// with lambda' correctly rounded (readings G9, G10).  Three-Pass: (mu) then (mu, 1 / sigma).
template <int A>
__device__ __forceinline__ float4 row_stats_of(int phase, float2 root, float mu) {
    if (A == kRecompute || A == kReload) {
        if (phase == 0) return make_float4(root.x, 0.0f, 0.0f, 0.0f);
        return make_float4(mu, __fdiv_rn(1.0f, root.x), root.x, 0.0f);
    }
    return make_float4(__fsub_rn(root.y, 1.0f), __fdiv_rn(0.5f, root.x), root.x, root.y);
}

__device__ __forceinline__ bool wait_flag(const unsigned* f, unsigned want, unsigned* err) {
    unsigned ns = 32;
    const unsigned long long t0 = globaltimer_ns();
    while (ld_acquire_gpu(f) != want) {
        __nanosleep(ns);
        ns = ns < 256 ? ns * 2 : ns;
        if (globaltimer_ns() - t0 > kWaitTimeoutNs) {  // never hang the GPU on a bug
            raise_abort(err, 1u);
            return false;
        }
    }
    return true;
}

// Watchdog-guarded mbarrier wait: false when the launch is being aborted (another role gave up,
// or this wait exceeded kWaitTimeoutNs; `bit` then records which wait).  A bug must never leave
// the GPU spinning: every role leaves its loop on an abort and the host sees the flags.
__device__ __forceinline__ bool wait_or_abort(uint64_t* bar, uint32_t parity, unsigned* err, unsigned bit) {
    if (mbar_try_parity(bar, parity)) return true;
    const unsigned long long t0 = globaltimer_ns();
    for (unsigned i = 1;; ++i) {
        if (mbar_try_parity(bar, parity)) return true;
        if ((i & 63u) == 0) {
            if (*reinterpret_cast<volatile unsigned*>(err)) return false;
            if (globaltimer_ns() - t0 > kWaitTimeoutNs) {
                raise_abort(err, bit);
                return false;
            }
        }
    }
}

// The same for a service warp that waits most of the time: it sleeps between polls, so that its
// polling does not take issue slots from the compute warps of its scheduler.
__device__ __forceinline__ bool wait_sleep_or_abort(uint64_t* bar, uint32_t parity, unsigned* err, unsigned bit) {
    if (mbar_try_parity(bar, parity)) return true;
    const unsigned long long t0 = globaltimer_ns();
    for (unsigned i = 1;; ++i) {
        __nanosleep(64);
        if (mbar_try_parity(bar, parity)) return true;
        if ((i & 63u) == 0) {
            if (*reinterpret_cast<volatile unsigned*>(err)) return false;
            if (globaltimer_ns() - t0 > kWaitTimeoutNs) {
                raise_abort(err, bit);
                return false;
            }
        }
    }
}

__device__ __forceinline__ bool aborted(unsigned* err) { return *reinterpret_cast<volatile unsigned*>(err) != 0; }

__device__ __forceinline__ void exit_and_reset(WsHeader* hdr) {
    __threadfence();
    const unsigned t = atomicAdd(&hdr->exit_ticket, 1u);
    if (t == gridDim.x - 1) {  // last CTA out resets the queue and advances the epoch
        hdr->counter = 0ull;
        hdr->exit_ticket = 0u;
        __threadfence();
        atomicAdd(&hdr->epoch, 1u);
    }
}

}  // namespace tp
