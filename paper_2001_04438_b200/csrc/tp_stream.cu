// Warp-specialised persistent kernel for 16-byte aligned rows (the fast path of every entry
// point).  One CTA per SM, three roles:
//
//   16 compute warps   execute commands from the producer in order.  A command names a stage
//                      and an operation (tp_ops.cuh) on the block in it; the warps copy their
//                      32 x 32 values into registers, compute, store outputs with 128-bit
//                      evict-first stores and hand per-warp results to the retire warp through
//                      a ring of part slots.  They never touch a global atomic or fence.
//   producer warp      takes items from the in-order work queue (chunks of 2, the next chunk's
//                      atomic in flight), starts a cp.async.bulk (TMA) copy of each item's block
//                      into a free stage, polls the row flags its items depend on (never
//                      blocking), and pushes commands as their inputs become available.
//   retire warp        publishes finished blocks in batches (one value per lane, one fence per
//                      batch) and runs the group / row reductions they complete (tp_ops.cuh).
//
// Two schedules:
//   hold    (Two-Pass, rows of 2..hold_max blocks): an item is one block; the block stays in
//           its stage between pass 1 (command P1) and pass 2 (command P2, pushed once the row's
//           pass 1 is released), so pass 2 re-reads it from shared memory, not from L2/HBM.
//   stream  (single-block rows, rows too long to hold, partial/finish, Three-Pass): an item is
//           one phase of one block (tp_sched.cuh decode_item); its stage is released as soon as
//           the values are in registers.
//
// Barriers: full[s] (count 1 + TMA bytes), empty[s] (count 16, one per compute warp when it is
// done reading the stage), cmd_full[c] (count 1) / cmd_empty[c] (count 16) for the command ring,
// pfull[r] (count 16) / pempty[r] (count 1) for the part ring.
// Deadlock freedom: items are handed out in increasing order; a command is pushed only when
// its inputs exist (no compute warp ever waits for a row); no role blocks on a row flag; so the
// smallest unfinished item always progresses.  In hold mode a CTA reserves an item only for a
// stage that is free or certain to free (its P2 pushed), one item per stage, so every reserved
// block gets staged; a row must fit in the CTAs' stages (hold_max = grid * S / 4 blocks), so the
// held blocks cannot all belong to the oldest unreleased row: some stage frees, the queue
// advances, and that row's remaining blocks get staged.
#include "tp_ops.cuh"

namespace tp {

constexpr int kProducerWarp = kWarps;
constexpr int kRetireWarp = kWarps + 1;
constexpr int kStreamThreads = kThreads + 64;
constexpr int kPartSlots = 8;
constexpr int kCmdSlots = 16;

template <typename In> struct Ring { static constexpr int S = 3; };   // 3 x 64 KB fp32
template <> struct Ring<uint16_t> { static constexpr int S = 6; };     // 6 x 32 KB bf16

enum CmdOp : int { kOpItem = 0, kOpP1 = 1, kOpP2 = 2, kOpExit = 3 };

struct StageMeta {
    long long item;
    Item it;
    int valid;
    unsigned mask;  // pass 2: per-warp clamp decisions of pass 1
    float4 stats;
};

struct Cmd {
    int op;
    int stage;
    unsigned parity;  // full[stage] parity of this use
};

struct PartSlot {
    long long item;
    Item it;
    float mu;
    Part part;
};

// 18 warps: 5 on some SM sub-partitions, whose 16K-register files then allow 96 per thread.
template <typename In, int A>
__global__ void __launch_bounds__(kStreamThreads, 1) stream_kernel(const KArgs a) {
    constexpr int P = AlgoTraits<A>::P;
    constexpr int V = InTraits<In>::V;
    constexpr int S = Ring<In>::S;
    constexpr int R = kPartSlots;
    constexpr int C = kCmdSlots;
    extern __shared__ __align__(128) unsigned char dsm[];
    __shared__ StageMeta meta[S];
    __shared__ PartSlot pslot[R];
    __shared__ Cmd cmds[C];
    __shared__ __align__(8) uint64_t full_bar[S];
    __shared__ __align__(8) uint64_t empty_bar[S];
    __shared__ __align__(8) uint64_t cfull_bar[C];
    __shared__ __align__(8) uint64_t cempty_bar[C];
    __shared__ __align__(8) uint64_t pfull_bar[R];
    __shared__ __align__(8) uint64_t pempty_bar[R];
    __shared__ unsigned s_epoch;

    pdl_wait_and_release();  // programmatic launch: the previous grid on the stream is complete
    publish_abort_word(a);
    WsHeader* hdr = reinterpret_cast<WsHeader*>(a.ws);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    In* stages = reinterpret_cast<In*>(dsm);
    const long long total = a.total_items;
    const bool hold = a.hold != 0;

    if (threadIdx.x == kProducerWarp * 32) {
        s_epoch = *reinterpret_cast<volatile unsigned*>(&hdr->epoch);
        for (int s = 0; s < S; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], kWarps);
        }
        for (int c = 0; c < C; ++c) {
            mbar_init(&cfull_bar[c], 1);
            mbar_init(&cempty_bar[c], kWarps);
        }
        for (int r = 0; r < R; ++r) {
            mbar_init(&pfull_bar[r], kWarps);
            mbar_init(&pempty_bar[r], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const unsigned want = s_epoch + 1u;

    if (warp == kProducerWarp) {
        // =============================================================== producer warp
        if (lane != 0) return;
        // development timeline (KArgs::prof): per CTA, globaltimer at start, at queue
        // exhaustion, at exit, when the first later-phase item was taken and when its row
        // statistics were first seen, in prof[16 + 5 * blockIdx.x + {0..4}]
        const unsigned long long tl_start = a.prof ? globaltimer_ns() : 0ull;
        unsigned long long tl_exh = 0, tl_p2 = 0, tl_rel = 0;
        const unsigned* row_ready = reinterpret_cast<const unsigned*>(a.ws + a.lay.row_ready);
        const In* x = static_cast<const In*>(a.x);
        const uint64_t pol_keep = policy_evict_last(), pol_drop = policy_evict_first();
        constexpr unsigned long long kChunk = 2;
        // stream mode: chunks of kChunk items, the next chunk's atomic in flight
        unsigned long long next = 0, end = 0, ahead = 0;
        if (!hold) {
            next = atomicAdd(&hdr->counter, kChunk);
            end = next + kChunk;
            ahead = atomicAdd(&hdr->counter, kChunk);  // result used one chunk later
        }
        bool exhausted = false;
        long long pushed = 0;
        // per stage, in registers: parity of the next use (bit s of use_par), state (2 bits: 0 free,
        // 1 busy until its empty barrier completes, 2 waiting for stats, 3 retired (hold mode:
        // its reservation was past the end)); the stages waiting for stats in issue order, oldest
        // in the low nibble of wq (wn entries): their commands are pushed in that order
        unsigned use_par = 0, st_bits = 0, wq = 0;
        int wn = 0;
        auto state_of = [&](int s) -> int { return (int)((st_bits >> (2 * s)) & 3u); };
        auto set_state = [&](int s, int v) { st_bits = (st_bits & ~(3u << (2 * s))) | ((unsigned)v << (2 * s)); };
        auto wait_stats = [&](int s) {  // stage s now waits for its row statistics
            set_state(s, 2);
            wq |= (unsigned)s << (4 * wn);
            ++wn;
        };
        // hold mode: each stage owns one reservation, taken when the stage is certain to free
        // without waiting on anything (at start, and when its P2 command is pushed).  A CTA
        // never reserves a block it cannot stage, so the oldest unreleased row always gets all
        // its blocks staged (a row must not wait on a block queued behind held stages).
        unsigned long long resv[S];
        if (hold)
            for (int s = 0; s < S; ++s) resv[s] = atomicAdd(&hdr->counter, 1ull);
        long long dec_item = -2;  // the last decoded stream item (the next one is usually its neighbour)
        Item dec_it{0, 0, 0};
        int64_t cached_row = -1;
        int cached_phase = -1;
        float4 cached_st = make_float4(0.f, 0.f, 0.f, 0.f);
        unsigned long long wait_t0 = 0;

        // development (KArgs::prof): producer cycle accounting, summed over CTAs into prof[8..13] =
        // chunk switches (waiting for the prefetched atomic), issue, command-slot waits, loop
        // passes without an issue, total, items issued
        unsigned long long ppc[6] = {0, 0, 0, 0, 0, 0};
        unsigned long long pfx[2] = {0, 0};  // proxy fence, expect_tx + bulk copy issue
        const unsigned long long ppc_start = a.prof ? clock64() : 0ull;
        auto take = [&]() -> long long {
            if (next == end) {
                const unsigned long long c0 = a.prof ? clock64() : 0ull;
                next = ahead;
                end = next + kChunk;
                ahead = atomicAdd(&hdr->counter, kChunk);
                if (a.prof) ppc[0] += clock64() - c0;
            }
            return (long long)next++;
        };

        auto push = [&](int op, int s, unsigned parity) {
            const int c = (int)(pushed % C);
            const unsigned long long c0 = a.prof ? clock64() : 0ull;
            if (pushed >= C && !wait_or_abort(&cempty_bar[c], (uint32_t)(((pushed / C) - 1) & 1), &hdr->error, 64u))
                return;
            if (a.prof) ppc[2] += clock64() - c0;
            cmds[c] = Cmd{op, s, parity};
            mbar_arrive(&cfull_bar[c]);
            ++pushed;
        };

        // statistics of the row phase an item depends on, if released (cached per row)
        auto stats_ready = [&](const Item& it, int dep_phase, float4* st) -> bool {
            if (!(it.row == cached_row && dep_phase == cached_phase) && a.shard_mu) {
                cached_st = shard_stats<A>(a, it.row, dep_phase);  // sharded Three-Pass phase
                cached_row = it.row;
                cached_phase = dep_phase;
            } else if (!(it.row == cached_row && dep_phase == cached_phase)) {
                // phase_only: the statistics are those a previous full launch left in the workspace
                if (!a.phase_only && ld_acquire_gpu(row_ready + it.row * 2 + dep_phase) != want) {
                    const unsigned long long now = globaltimer_ns();
                    if (wait_t0 == 0) wait_t0 = now;
                    if (now - wait_t0 <= kWaitTimeoutNs) return false;
                    raise_abort(&hdr->error, 1u);  // never hang the GPU on a bug
                }
                if (a.prof && tl_rel == 0) tl_rel = globaltimer_ns();
                cached_st = __ldcg(reinterpret_cast<const float4*>(a.ws + a.lay.row_stats) + it.row * 2 + dep_phase);
                cached_row = it.row;
                cached_phase = dep_phase;
            }
            wait_t0 = 0;
            *st = cached_st;
            return true;
        };

        // push the commands whose statistics are now available, oldest item first
        auto poll = [&]() {
            while (wn > 0) {
                const int best = (int)(wq & 15u);
                const Item it = meta[best].it;
                float4 st;
                if (!stats_ready(it, hold ? 0 : it.phase - 1, &st)) return;
                meta[best].stats = st;
                meta[best].mask = (A == kTwoPass && st.z != 0.0f)
                                      ? __ldcg(reinterpret_cast<const unsigned*>(a.ws + a.lay.block_clamp) +
                                               it.row * a.nb + it.blk)
                                      : 0u;
                wq >>= 4;
                --wn;
                set_state(best, 1);
                push(hold ? kOpP2 : kOpItem, best, ((use_par >> best) & 1u) ^ 1u);
                if (hold) resv[best] = atomicAdd(&hdr->counter, 1ull);  // consumed when the stage frees
            }
        };

        auto issue = [&](int s, long long item) {
            Item it;
            if (hold || a.phase_only) {  // one item per block: (row, blk)
                const uint32_t u = (uint32_t)item, nb = (uint32_t)a.nb;
                it.phase = hold ? 0 : a.phase_only - 1;  // hold: pass 1 then pass 2 on the same stage
                it.row = u / nb;
                it.blk = u - (u / nb) * nb;
                // hold: pass 2 backwards; one phase alone: odd phases backwards (each phase
                // starts where the previous one ended, the L2-resident end)
                if (hold ? it.phase > 0 : (it.phase & 1)) it.blk = a.nb - 1 - it.blk;
            } else if (item == dec_item + 1 && (uint64_t)item % (uint64_t)a.nb != 0) {
                it = dec_it;  // the next block of the same (row, phase) unit (decode_item's direction)
                it.blk += (A == kFinish || it.phase > 0) ? -1 : 1;
            } else {
                it = decode_item<A>(item, a.rows, a.nb, a.L);
            }
            if (!hold && !a.phase_only) dec_item = item, dec_it = it;
            const int64_t e0 = it.blk * kBlockElems;
            const int valid = (int)min((int64_t)kBlockElems, a.cols - e0);
            meta[s].item = item;
            meta[s].it = it;
            meta[s].valid = valid;
            const unsigned parity = (use_par >> s) & 1u;
            use_par ^= 1u << s;
            if (A == kReload && it.phase == 2) {  // Reload's pass 3 reads Y, not X: no copy
                mbar_arrive(&full_bar[s]);
            } else {
                const uint32_t bytes = (uint32_t)valid * (uint32_t)sizeof(In);
                // evict_last for blocks a later pass re-reads: the interleaved schedule's early
                // phases, the partial (the finish follows), a sharded Three-Pass phase but its last
                const bool keep = !hold && (a.phase_only ? (a.shard_mu || a.shard_out) && it.phase < P - 1
                                                         : ((P > 1 && it.phase < P - 1) || A == kPartial));
                In* dst = stages + (size_t)s * kBlockElems;
                const unsigned long long f0 = a.prof ? clock64() : 0ull;
                // (no proxy fence: the stage's previous contents were only read, and those reads
                // are ordered before this copy by its empty barrier)
                const unsigned long long f1 = a.prof ? clock64() : 0ull;
                mbar_arrive_expect_tx(&full_bar[s], bytes);
                if (a.l2_hints) tma_load_1d(dst, x + it.row * a.cols + e0, bytes, &full_bar[s], keep ? pol_keep : pol_drop);
                else tma_load_1d_nohint(dst, x + it.row * a.cols + e0, bytes, &full_bar[s]);
                if (a.prof) pfx[0] += f1 - f0, pfx[1] += clock64() - f1;
            }
            if (A == kFinish) {
                if (it.row != cached_row) {
                    cached_st = finish_stats(a, it.row);
                    cached_row = it.row;
                }
                meta[s].stats = cached_st;
                meta[s].mask = finish_mask(a, cached_st, it.row, it.blk);  // the partial's clamp decisions
            }
            if (hold) {
                wait_stats(s);  // P1 now, P2 once the row is released
                push(kOpP1, s, parity);
            } else if (item_needs_stats<A>(it) && A != kFinish) {
                if (a.prof && tl_p2 == 0) tl_p2 = globaltimer_ns();
                wait_stats(s);
                poll();
            } else {
                set_state(s, 1);
                push(kOpItem, s, parity);
            }
        };

        if (A == kFinish && a.mailbox) finish_wait(a);  // fused NVLink exchange: the peers' pairs
        for (unsigned pass = 0;; ++pass) {
            // watchdog: every role leaves.  Polled every 64 passes: the flag shares the header
            // with the work-queue counter every producer's atomics hit
            if ((pass & 63u) == 63u && aborted(&hdr->error)) return;
            if (wn > 0) poll();
            bool busy = false, issued_now = false;
            for (int s = 0; s < S; ++s) {
                if (state_of(s) == 1 && mbar_test_parity(&empty_bar[s], ((use_par >> s) & 1u) ^ 1u)) set_state(s, 0);
                if (hold) {
                    if (state_of(s) == 0) {
                        if (resv[s] >= (unsigned long long)total) set_state(s, 3);
                        else issue(s, (long long)resv[s]);
                    }
                    busy |= state_of(s) != 3;
                    continue;
                }
                if (state_of(s) == 0 && !exhausted) {
                    const long long item = take();
                    if (item >= total) {
                        exhausted = true;
                        if (a.prof) tl_exh = globaltimer_ns();
                    } else {
                        const unsigned long long c0 = a.prof ? clock64() : 0ull;
                        issue(s, item);
                        if (a.prof) ppc[1] += clock64() - c0, ppc[5] += 1;
                        issued_now = true;
                    }
                }
                busy |= state_of(s) != 0;
            }
            if ((hold || exhausted) && !busy) break;
            if (a.prof && !issued_now) ppc[3] += 1;

        }
        push(kOpExit, 0, 0);
        if (!hold && ahead == ~0ull) hdr->error |= 2u;  // consume the last prefetch before leaving
        if (a.prof) {
            ppc[4] = clock64() - ppc_start;
            for (int i = 0; i < 6; ++i) atomicAdd(&a.prof[8 + i], ppc[i]);
            atomicAdd(&a.prof[14], pfx[0]);
            atomicAdd(&a.prof[15], pfx[1]);
            unsigned long long* t = a.prof + 16 + 5 * blockIdx.x;
            t[0] = tl_start;
            t[1] = tl_exh;
            t[2] = globaltimer_ns();
            t[3] = tl_p2;
            t[4] = tl_rel;
        }
        exit_and_reset(hdr);
    } else if (warp == kRetireWarp) {
        // =============================================================== retire warp
        for (long long seq = 0;;) {
            int n = 0;
            if (lane == 0) {
                if (wait_or_abort(&pfull_bar[seq % R], (uint32_t)((seq / R) & 1), &hdr->error, 32u)) {
                    n = 1;
                    while (n < R && mbar_test_parity(&pfull_bar[(seq + n) % R], (uint32_t)(((seq + n) / R) & 1))) ++n;
                }
            }
            n = __shfl_sync(0xffffffffu, n, 0);
            if (n == 0) break;  // aborted
            const bool have = lane < n;
            const PartSlot* ps = &pslot[(seq + lane) % R];
            const long long item = have ? ps->item : total;
            const unsigned stop = __ballot_sync(0xffffffffu, have && item >= total);
            const int m = stop ? __ffs(stop) - 1 : n;  // slots before the sentinel
            Item it{0, 0, 0};
            float2 val = make_float2(0.f, 0.f);
            float mu = 0.f;
            bool mine = false;
            if (lane < m) {
                it = ps->it;
                mu = ps->mu;
                mine = item_retires<A>(it);
                if (mine) val = block_value<A>(a, it, ps->part);
            }
            retire_batch<A>(a, mine, it, val, mu, want);
            __syncwarp();
            if (lane < m) mbar_arrive(&pempty_bar[(seq + lane) % R]);
            seq += m;
            if (stop) break;
        }
    } else {
        // =============================================================== compute warps
        long long pseq = 0;  // part slots used
        // development (KArgs::prof): compute warp cycle accounting, summed over CTAs into
        // prof[0..7] = command wait, data wait, part-slot wait, pass-1 ops, later-phase ops,
        // total, pass-1 blocks, later-phase blocks (warp 0 of each CTA)
        const bool pc_on = a.prof != nullptr && warp == 0;
        unsigned long long pc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const unsigned long long pc_start = pc_on ? clock64() : 0ull;
        unsigned long long pt = pc_start;
        auto lap = [&](int slot) {
            if (pc_on) {
                const unsigned long long now = clock64();
                pc[slot] += now - pt;
                pt = now;
            }
        };
        for (long long c = 0;; ++c) {
            const int cs = (int)(c % C);
            if (!wait_or_abort(&cfull_bar[cs], (uint32_t)((c / C) & 1), &hdr->error, 8u)) break;
            lap(0);
            const Cmd cmd = cmds[cs];
            __syncwarp();
            if (lane == 0) mbar_arrive(&cempty_bar[cs]);
            const int s = cmd.stage;
            if (cmd.op == kOpP2) {  // hold mode, pass 2 on the held block; no part slot
                const Item it = meta[s].it;  // read everything before the stage is released
                const int valid = meta[s].valid;
                const float4 st = meta[s].stats;
                const bool my_clamp = ((meta[s].mask >> warp) & 1u) != 0;
                BlockVals v;
                load_stage<In>(stages + (size_t)s * kBlockElems, v);
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty_bar[s]);
                op_pass2<V>(v, st, my_clamp, a.y + it.row * a.cols + it.blk * kBlockElems, valid, true);
                continue;
            }
            const int r = (int)(pseq % R);
            if (pseq >= R && !wait_or_abort(&pempty_bar[r], (uint32_t)(((pseq / R) - 1) & 1), &hdr->error, 16u)) break;
            ++pseq;
            lap(2);
            PartSlot& ps = pslot[r];
            if (cmd.op == kOpExit) {  // pass the end on to the retire warp
                if (warp == 0 && lane == 0) ps.item = total;
                __syncwarp();
                if (lane == 0) mbar_arrive(&pfull_bar[r]);
                break;
            }
            if (!wait_or_abort(&full_bar[s], cmd.parity, &hdr->error, 4u)) break;
            lap(1);
            const long long item = meta[s].item;  // read everything before the stage is released
            const Item it = meta[s].it;
            const int valid = meta[s].valid;
            const float4 st = meta[s].stats;
            const bool my_clamp = ((meta[s].mask >> warp) & 1u) != 0;
            float* yb = a.y ? a.y + it.row * a.cols + it.blk * kBlockElems : nullptr;
            BlockVals v;
            if (!(A == kReload && it.phase == 2)) load_stage<In>(stages + (size_t)s * kBlockElems, v);
            if (cmd.op == kOpItem) {  // stream mode: the values are in registers, free the stage
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty_bar[s]);
            }

            if constexpr (A == kFused) {
                op_pass1<V>(v, valid, ps.part);
                asm volatile("bar.sync 1, %0;" ::"r"(kThreads) : "memory");  // compute warps only
                op_fused_tail<V>(v, ps.part, yb, valid, true);
            } else if constexpr (A == kTwoPass || A == kPartial) {
                if (it.phase == 0) op_pass1<V>(v, valid, ps.part);  // kOpP1 (hold) or stream pass 1
                else op_pass2<V>(v, st, my_clamp, yb, valid, true);
            } else if constexpr (A == kFinish) {
                op_pass2<V>(v, st, my_clamp, yb, valid, true);
            } else {
                if (it.phase == 0) op_max<V>(v, valid, ps.part);
                else if (it.phase == 1) op_expsum<V, A == kReload>(v, valid, st.x, ps.part, yb, true);
                else if (A == kRecompute) op_out_recompute<V>(v, st, yb, valid, true);
                else op_out_reload(st, yb, valid, true);
            }
            if (warp == 0 && lane == 0) {
                ps.item = item;
                ps.it = it;
                ps.mu = st.x;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&pfull_bar[r]);
            if (pc_on) {
                lap(it.phase == 0 ? 3 : 4);
                ++pc[it.phase == 0 ? 6 : 7];
            }
        }
        if (pc_on && lane == 0) {
            pc[5] = clock64() - pc_start;
            for (int i = 0; i < 8; ++i) atomicAdd(&a.prof[i], pc[i]);
        }
    }
}

template <typename In, int A>
cudaError_t launch_stream(KArgs a, const LaunchOpts& o, cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    auto kern = stream_kernel<In, A>;
    constexpr int S = Ring<In>::S;
    const size_t dyn = (size_t)S * kBlockElems * sizeof(In);
    static DevCache configured[kMaxDevices];
    if (!configured[dev].load(std::memory_order_acquire)) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        configured[dev].store(1, std::memory_order_release);
    }
    const int64_t resident = device_sms(dev);  // one CTA per SM
    int64_t grid = o.grid_ctas > 0 ? o.grid_ctas : resident;
    if (grid > resident) grid = resident;
    // hold mode: Two-Pass rows of several blocks that fit the grid's stages four times over
    a.hold = (A == kTwoPass && o.schedule == 2 && a.nb >= 2 && a.nb * 4 <= grid * S && !a.phase_only) ? 1 : 0;
    if (a.hold || a.phase_only) a.total_items = a.rows * a.nb;
    if (grid > a.total_items) grid = a.total_items;
    if (grid < 1) grid = 1;
    // stream mode: items a CTA holds between hand-out and retirement (its stages, the prefetched
    // queue chunks and the part-slot backlog; measured: C4 gains up to L ~ 50 rows)
    a.L = lookahead_rows(a, grid, S + 12, o);
    last_plan() = Plan{2, A, grid, 0, a.L, a.hold};
    // programmatic dependent launch (the kernel waits for the previous grid before touching
    // memory): the launch overlaps the previous kernel's tail (development override TP_PDL=0)
    static const int pdl = dev_env_int("TP_PDL", 1);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kStreamThreads);
    cfg.dynamicSmemBytes = dyn;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

#define TP_INSTANTIATE(IN)                                                                     \
    template cudaError_t launch_stream<IN, kTwoPass>(KArgs, const LaunchOpts&, cudaStream_t);   \
    template cudaError_t launch_stream<IN, kPartial>(KArgs, const LaunchOpts&, cudaStream_t);   \
    template cudaError_t launch_stream<IN, kRecompute>(KArgs, const LaunchOpts&, cudaStream_t); \
    template cudaError_t launch_stream<IN, kReload>(KArgs, const LaunchOpts&, cudaStream_t);    \
    template cudaError_t launch_stream<IN, kFused>(KArgs, const LaunchOpts&, cudaStream_t);     \
    template cudaError_t launch_stream<IN, kFinish>(KArgs, const LaunchOpts&, cudaStream_t);
TP_INSTANTIATE(float)
TP_INSTANTIATE(uint16_t)

}  // namespace tp
