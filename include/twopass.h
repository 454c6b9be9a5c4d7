/*
 * twopass.h — C ABI of libtwopass.so, a B200 (sm_100a) implementation of
 * "The Two-Pass Softmax Algorithm" (Dukhan & Ablavatski, arXiv 2001.04438).
 *
 * Operation (all entry points): row-wise softmax of a row-major matrix,
 *     y[r][i] = e^{x[r][i]} / sum_k e^{x[r][k]}                (§1)
 * computed by Alg. 3 SoftmaxTwoPass (§4): pass 1 reads each row
 * once, turns every x into an extended-exponent pair (m, n) with e^x = m 2^n
 * (ExtExp) and reduces the pairs with max-exponent
 * rescaling to (m_sum, n_sum); pass 2 re-reads the row and
 * writes y = m * lambda_sum * 2^{n - n_sum} with lambda_sum = 1/m_sum
 * (PAPER.md:164-168).  No max pass; no overflow for any finite input.
 * The softmax3_* entry points are the in-house Three-Pass comparators
 * (Alg. 1 Recompute; Alg. 2 Reload).
 *
 * Conventions shared by every entry point
 *   Layout     x: rows x cols, row-major, contiguous, row stride = cols elements.
 *              y: rows x cols fp32, same layout.  bf16 inputs are raw bf16 bit
 *              patterns (uint16_t), converted exactly to fp32; arithmetic and
 *              output are fp32.
 *   Memory     x, y, pairs: DEVICE pointers (cudaMalloc / torch), owned by the
 *              caller; the library never frees them.  Any alignment is accepted;
 *              16-byte aligned rows (cols % 4 == 0 fp32, % 8 == 0 bf16, 16-byte
 *              aligned bases) use 128-bit loads/stores.
 *   Aliasing   fp32 entry points allow y == x exactly (in place); any partial
 *              overlap of x and y is rejected.  bf16 entry points reject overlap.
 *   Streams    Enqueue-only: the call returns after launching on `stream`
 *              (0 = legacy default stream) without synchronising.  Execution
 *              errors surface at the caller's next synchronisation.  Some kernels
 *              are programmatic dependent launches: they may be scheduled while
 *              the stream's previous kernel runs but touch no memory before it
 *              has completed, so stream order is kept.
 *   Workspace  Entry points without a workspace argument use one internal
 *              per-device workspace (allocated, zero-filled and grown on first
 *              use; growth synchronises the device).  Calls that use it must not
 *              run concurrently on different streams of one device; use the _ex
 *              variants with caller-owned workspaces for that and for CUDA-graph
 *              capture.
 *   Accuracy   Per element, against the exact softmax o: |y - o| <= 2e-5 o for
 *              o >= FLT_MIN, |y - o| <= 1e-37 below (BASELINE.json north_star),
 *              for finite |x| <= 2^21 (reading G11; larger magnitudes
 *              are clamped to +-2^21, NaN is treated as -2^21).
 *   Determinism Results are bitwise reproducible and independent of grid size,
 *              stream, alignment and (for the partial/finish path with a
 *              power-of-two world and block-aligned equal chunks) of the number
 *              of ranks (reading G8).
 *   Status     0 TP_OK; 1 TP_EINVAL (null pointer, rows < 1 or cols < 1, partial
 *              x/y overlap, world < 1, workspace too small); 2 TP_ECUDA (launch
 *              or allocation error: see softmax_last_cuda_error()); 3 TP_ENODEV
 *              (no CUDA device); 4 TP_EWATCHDOG (an EARLIER launch on this device
 *              gave up a wait after 4 s, or a mailbox wait timed out, and its
 *              outputs are invalid: reported once, by the first call after the
 *              abort became visible to the host; the library has reset its state
 *              and the next call runs normally).  Nothing is launched when the
 *              status is not 0.
 */
#ifndef TWOPASS_H
#define TWOPASS_H

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { TP_OK = 0, TP_EINVAL = 1, TP_ECUDA = 2, TP_ENODEV = 3, TP_EWATCHDOG = 4 };

/* Algorithm and input-dtype selectors of the _ex entry points. */
enum { TP_ALGO_TWO_PASS = 0, TP_ALGO_THREE_PASS_RECOMPUTE = 2, TP_ALGO_THREE_PASS_RELOAD = 3 };
enum { TP_IN_F32 = 0, TP_IN_BF16 = 1 };

/* ---- Two-Pass softmax (Alg. 3) -------------------------- */
int softmax_f32(const float* x, float* y, int64_t rows, int64_t cols, cudaStream_t stream);
int softmax_bf16_f32(const uint16_t* x, float* y, int64_t rows, int64_t cols, cudaStream_t stream);

/* ---- Three-Pass comparators: Recompute (Alg. 1) and Reload
 *      (Alg. 2), same polynomial and range reduction as ExtExp
 *       plus reconstruction with flush below 2^-126. */
int softmax3_recompute_f32(const float* x, float* y, int64_t rows, int64_t cols, cudaStream_t stream);
int softmax3_reload_f32(const float* x, float* y, int64_t rows, int64_t cols, cudaStream_t stream);
int softmax3_recompute_bf16_f32(const uint16_t* x, float* y, int64_t rows, int64_t cols, cudaStream_t stream);
int softmax3_reload_bf16_f32(const uint16_t* x, float* y, int64_t rows, int64_t cols, cudaStream_t stream);

/* ---- Split Two-Pass for sharded rows (multi-GPU, BASELINE.json north_star) ----
 * partial: pass 1 of Alg. 3 over a chunk of every row, reduced
 *   to one pair per row: pair_out[2r] = m_sum, pair_out[2r+1] = n_sum (device,
 *   rows x 2 fp32).  The chunk's pair represents sum_i e^{x_i} = m_sum 2^{n_sum}.
 * finish: merges `world` partials per row (pairs: device, world x rows x 2 fp32,
 *   rank-major: pairs[(w*rows + r)*2 + {0,1}]) with a balanced tree over rank index,
 *   computes lambda_sum = 1/m_sum and runs pass 2
 *   over the local chunk x -> y.  With world == 1 the result equals softmax_f32's
 *   bit for bit.                                                                */
int softmax_f32_partial(const float* x, int64_t rows, int64_t cols, float* pair_out, cudaStream_t stream);
int softmax_bf16_partial(const uint16_t* x, int64_t rows, int64_t cols, float* pair_out, cudaStream_t stream);
int softmax_f32_finish(const float* x, float* y, int64_t rows, int64_t cols, const float* pairs, int world,
                       cudaStream_t stream);
int softmax_bf16_f32_finish(const uint16_t* x, float* y, int64_t rows, int64_t cols, const float* pairs,
                            int world, cudaStream_t stream);

/* ---- Three-Pass comparators for sharded rows (multi-GPU Alg. 1 / Alg. 2) ----
 * The comparators need TWO exchanges per call where the Two-Pass needs one:
 *   max_partial : pass 1 over the local chunk -> max_out[r] (device, rows fp32)
 *   -> gather every rank's maxima: maxes, device, world x rows, rank-major
 *   sum_partial : mu = max over ranks; pass 2 (PAPER.md:93-95 / 111-117) over the local chunk ->
 *                 sum_out[r] = sum of Exp(x - mu) (device, rows); Reload (algo 3) also writes
 *                 y = Exp(x - mu) (y may be NULL for Recompute)
 *   -> gather every rank's sums: sums, device, world x rows, rank-major
 *   finish      : sigma = canonical tree over rank index of the sums (reading G8), lambda =
 *                 1/sigma; pass 3 (PAPER.md:96-98 / 119-121): y = lambda Exp(x - mu) (Recompute,
 *                 re-reads x) or y = lambda y (Reload, re-reads y)
 * algo: TP_ALGO_THREE_PASS_RECOMPUTE or TP_ALGO_THREE_PASS_RELOAD (the same for all three calls).
 * With world == 1 (maxes / sums = the chunk's own results) the outputs equal softmax3_*'s bit for
 * bit; with a power-of-two world and equal chunks that are power-of-two runs of 16384-element
 * blocks, bitwise those of one GPU.  Workspace as for softmax_ex (NULL, 0 = internal; one per
 * concurrent stream).  Asynchronous; statuses as above. */
int softmax3_max_partial_ex(int in_dtype, const void* x, int64_t rows, int64_t cols, float* max_out, void* workspace,
                            size_t workspace_bytes, cudaStream_t stream);
int softmax3_sum_partial_ex(int algo, int in_dtype, const void* x, float* y, int64_t rows, int64_t cols,
                            const float* maxes, int world, float* sum_out, void* workspace, size_t workspace_bytes,
                            cudaStream_t stream);
int softmax3_finish_ex(int algo, int in_dtype, const void* x, float* y, int64_t rows, int64_t cols, const float* maxes,
                       const float* sums, int world, void* workspace, size_t workspace_bytes, cudaStream_t stream);

/* ---- one-sided pair exchange over NVLink (rank merge without a collective) --
 * A mailbox (device memory of tp_mailbox_bytes(world, rows) bytes, owned by its rank, ZERO-
 * FILLED once before first use) is double-buffered by epoch parity h = epoch & 1: bytes
 * [256 h, 256 h + 4 world) one uint32 flag per rank, bytes [512, 516) an error word (bit r:
 * waiting for rank r timed out), and from byte tp_mailbox_pairs_offset(world, rows, epoch)
 * (= 1024 + h * 8 * world * rows) the pairs float[world][rows][2] of that epoch (rank-major,
 * the layout softmax_f32_finish takes).  world <= 56.  Two halves make reuse safe: a rank
 * pushes epoch e + 2 only after its finish of e + 1, which waited for every rank's push of
 * e + 1, issued by each rank after its own finish of e had read half e & 1.
 * tp_pairs_push: after softmax_*_partial on rank `rank`, stores its rows pairs (device) into
 *   slot `rank` of every mailbox listed in peer_mailboxes (DEVICE array of world pointers,
 *   entry p = rank p's mailbox mapped into this process: the local one, or one opened with
 *   tp_ipc_open), then release-stores `epoch` into flag `rank` of each (system scope).
 * tp_pairs_wait: on the local mailbox, waits until every flag equals `epoch` (acquire,
 *   system scope), or timeout_ns elapsed (then sets the error word; outputs are undefined).
 * Both asynchronous on `stream`; use a new epoch (e.g. 1, 2, ...) per exchange, the same on
 * all ranks.  Then softmax_*_finish(x, y, rows, cols, mailbox + tp_mailbox_pairs_offset(...),
 * world, ...).
 * Sequence per rank: partial -> push -> wait -> finish; no NCCL, no host synchronisation.   */
size_t tp_mailbox_bytes(int world, int64_t rows);
size_t tp_mailbox_pairs_offset(int world, int64_t rows, unsigned epoch); /* 0 on bad arguments */
int tp_pairs_push(const float* pairs, int64_t rows, void* const* peer_mailboxes, int rank, int world,
                  unsigned epoch, cudaStream_t stream);
int tp_pairs_wait(const void* mailbox, int world, unsigned epoch, uint64_t timeout_ns, cudaStream_t stream);
/* CUDA IPC plumbing for the mailboxes (one process per GPU): tp_ipc_get_handle gives the
 * 64-byte handle of the device allocation containing dev_ptr (made by this process, e.g. a
 * caching-allocator segment) and dev_ptr's byte offset in it; tp_ipc_open maps a peer
 * process's (handle, offset) into this process (peer access enabled lazily) and returns the
 * pointer; tp_ipc_close unmaps a pointer tp_ipc_open returned.                              */
int tp_ipc_get_handle(const void* dev_ptr, void* handle64, uint64_t* offset);
int tp_ipc_open(const void* handle64, uint64_t offset, void** dev_ptr);
int tp_ipc_close(void* dev_ptr);

/* ---- explicit-workspace / tuning variants ----------------------------------
 * workspace: device memory of at least softmax_workspace_bytes(rows, cols) bytes (it includes
 *   a second layout for the tail rows a cluster launch may hand to a concurrent launch),
 *   ZERO-FILLED before its first use; the kernels leave it reusable.  One
 *   workspace must not be used by two launches running concurrently.
 * opts: may be NULL.  grid_ctas = persistent grid size (0 = one resident wave;
 *   larger values are clamped to it); lookahead_rows = rows of pass 1 kept ahead of
 *   pass 2 (0 = automatic); force_persistent = two-phase schedule even for rows that
 *   fit one block; disable_tma = load blocks with 128-bit global loads instead of TMA
 *   bulk copies into shared memory; schedule = TP_SCHED_AUTO (0), TP_SCHED_STREAM (1:
 *   a persistent grid shares every row, pass-2 blocks are re-read from L2/HBM),
 *   TP_SCHED_HOLD (2: as STREAM, but Two-Pass rows of a few blocks stay staged in shared
 *   memory between the passes) or TP_SCHED_CLUSTER (3: rows of 2..256 blocks, one
 *   thread-block cluster per row, the row's block values exchanged through distributed
 *   shared memory, the re-reads from shared memory / L2; AUTO picks it for the Two-Pass
 *   when the cluster's L2 working set fits; for the Three-Pass comparators only on request);
 *   a schedule that does not apply falls back to STREAM;
 *   cluster_size = CTAs per row for TP_SCHED_CLUSTER (0 = automatic; 1, 2, 4, 8 or 16).
 *   Results do not depend on any of these (bit-identical outputs). */
#define TP_SCHED_AUTO 0
#define TP_SCHED_STREAM 1
#define TP_SCHED_HOLD 2
#define TP_SCHED_CLUSTER 3
#define TP_SCHED_SMALL 4  /* rows of 1..3 blocks: one CTA per row, the row staged in shared
                             memory (AUTO picks it for at most 2 x SMs such rows) */
#define TP_SCHED_PHASE 5  /* a few very long rows (Two-Pass: at most 8 rows; partial / finish:
                             any): one CTA per SM taking all pass-1 blocks, then all pass-2
                             blocks, from an in-order queue, no command ring (AUTO picks it for
                             the Two-Pass from ~100 blocks per SM, the partial from ~48) */
#define TP_SCHED_RESIDENT 6  /* Two-Pass rows of 4..64 blocks whose share fits shared memory
                                (bf16: <= 7 blocks per CTA, fp32: <= 3): a group of CTAs per
                                row stages its whole share, exchanges block values through the
                                workspace, and runs pass 2 on the staged blocks (the row is read
                                from HBM once); cluster_size = CTAs per row (0 = automatic;
                                AUTO picks it for bf16 rows of 4..64 blocks, one block per CTA) */
typedef struct {
    int64_t grid_ctas;
    int64_t lookahead_rows;
    int force_persistent;
    int disable_tma;
    int schedule;
    int cluster_size;
} softmax_opts;

size_t softmax_workspace_bytes(int64_t rows, int64_t cols);
int softmax_ex(int algo, int in_dtype, const void* x, float* y, int64_t rows, int64_t cols, void* workspace,
               size_t workspace_bytes, const softmax_opts* opts, cudaStream_t stream);
int softmax_partial_ex(int in_dtype, const void* x, int64_t rows, int64_t cols, float* pair_out, void* workspace,
                       size_t workspace_bytes, const softmax_opts* opts, cudaStream_t stream);
/* softmax_finish_ex: as softmax_f32_finish / softmax_bf16_f32_finish on a caller workspace
 *   (NULL with 0 bytes = the internal one).  Pass the workspace the chunk's partial call used:
 *   the partial leaves there, per block, the warps whose pass 1 ran on clamped values (reading
 *   G11, |x| > 2^21), and the finish replays exactly those choices, so outputs are bitwise
 *   those of one GPU for any input.  With another workspace only elements outside the accuracy
 *   domain (|x| > 2^21) can differ.  A workspace must not be used by two launches running
 *   concurrently. */
int softmax_finish_ex(int in_dtype, const void* x, float* y, int64_t rows, int64_t cols, const float* pairs,
                      int world, void* workspace, size_t workspace_bytes, const softmax_opts* opts,
                      cudaStream_t stream);

/* ---- fused one-sided exchange (pass 1 + rank merge a7 without a collective
 * library or extra launches; mailboxes as for tp_pairs_push / tp_pairs_wait above) ----------
 * softmax_partial_push_ex: pass 1 of Alg. 3 over this rank's chunk of each
 *   row, as softmax_partial_ex; inside the same kernel, the thread that finishes a row's
 *   pair stores it into slot `rank` of every mailbox in peer_mailboxes (DEVICE array of world
 *   pointers, as tp_pairs_push) and, once all `rows` pairs are stored and fenced system-wide,
 *   release-stores `epoch` (>= 1, new per exchange) into flag `rank` of every mailbox.
 *   pair_out (device, rows x 2) also receives the pairs when not NULL.
 * softmax_finish_mailbox_ex: as softmax_finish_ex with pairs = this epoch's half of the mailbox, except
 *   that the kernel itself first waits (acquire, system scope) until the world flags of the
 *   LOCAL mailbox equal `epoch`; a flag missing for timeout_ns sets its rank's bit in the
 *   mailbox error word and watchdog bit 0 (outputs then undefined; nothing hangs; the next
 *   call on the device returns TP_EWATCHDOG).  workspace: as softmax_finish_ex (the one
 *   softmax_partial_push_ex used).
 * Sequence per rank: partial_push -> finish_mailbox, two launches, no NCCL, no host
 * synchronisation.  Results are bit-identical to partial -> all_gather -> finish.  The epoch is
 * a launch argument: a captured CUDA graph replays the same epoch, so a graph must be captured
 * per epoch (or the mailboxes zeroed between replays) for its waits to mean anything.
 * TP_EINVAL: bad sizes / pointers, world outside 1..56, rank outside [0, world), epoch 0,
 * mailbox not 16-byte aligned.  Asynchronous. */
int softmax_partial_push_ex(int in_dtype, const void* x, int64_t rows, int64_t cols, void* const* peer_mailboxes,
                            int rank, int world, unsigned epoch, float* pair_out, void* workspace,
                            size_t workspace_bytes, const softmax_opts* opts, cudaStream_t stream);
int softmax_finish_mailbox_ex(int in_dtype, const void* x, float* y, int64_t rows, int64_t cols, const void* mailbox,
                              int world, unsigned epoch, unsigned long long timeout_ns, void* workspace,
                              size_t workspace_bytes, const softmax_opts* opts, cudaStream_t stream);

/* ---- end-to-end call on HOST buffers ---------------------------------------
 * hx, hy: HOST pointers (pinned memory gives full PCIe bandwidth).  Copies x to
 * the current device, runs softmax_f32 / softmax_bf16_f32, copies y back and
 * returns when hy is filled (synchronous).  Row slabs are pipelined over two
 * streams so host->device copies, kernels and device->host copies overlap.
 * Device staging memory is cached per device between calls.                   */
int softmax_f32_host(const float* hx, float* hy, int64_t rows, int64_t cols);
int softmax_bf16_f32_host(const uint16_t* hx, float* hy, int64_t rows, int64_t cols);

/* Asynchronous form of the host-buffer call (throughput: consecutive calls overlap, one call's
 * host->device copies with the previous call's device->host copies, the two PCIe directions at
 * once).  Enqueues the copies and kernels of one call on the library's internal streams of the
 * current device and returns; *ticket identifies the call.  Submitted calls alternate between two
 * internal staging slots (device memory for x and y of one call each, cached), so at most two run
 * at a time; a third submission queues behind the first on its slot.
 * in_dtype: TP_IN_F32 / TP_IN_BF16.  hx, hy: HOST pointers (pinned for full bandwidth) that must
 * stay valid and untouched until softmax_host_wait(ticket) returns.  Results are bit-identical to
 * softmax_f32_host.  Returns TP_EINVAL for bad arguments or a NULL ticket pointer.              */
int softmax_host_submit(int in_dtype, const void* hx, float* hy, int64_t rows, int64_t cols,
                        unsigned long long* ticket);
/* Blocks until the call `ticket` (and every earlier call on its slot) has completed and hy is
 * filled.  A ticket more than 15 submissions old on its device is rejected (TP_EINVAL).       */
int softmax_host_wait(unsigned long long ticket);

/* ---- status ---------------------------------------------------------------- */
/* What the last launch issued by this host thread ran (diagnostics; no device work):
 * kernel = 1 general (any alignment), 2 stream (persistent grid), 3 cluster (one
 * thread-block cluster per row), 4 small (one CTA per row of <= 3 blocks), 5 phase (static
 * schedule of a few long rows; hold = its stages); variant = the kernel's operation (0 Two-Pass, 1 partial,
 * 2 Recompute, 3 Reload, 4 single-block rows, 5 finish); grid_ctas; cluster_size (kernel 3);
 * lookahead_rows (kernel 1/2; kernel 3: rows handed to a concurrent side launch on the SMs
 * the clusters leave idle, 0 if none); hold (kernel 2: blocks kept staged between the passes;
 * kernel 3: half-stages of the pass-1 pool).  Returns TP_EINVAL for a NULL pointer. */
typedef struct {
    int kernel;
    int variant;
    int64_t grid_ctas;
    int cluster_size;
    int64_t lookahead_rows;
    int hold;
} softmax_plan;
int softmax_last_plan(softmax_plan* out);

const char* softmax_status_str(int status);
int softmax_last_cuda_error(void); /* cudaError_t of the last TP_ECUDA on this thread */
/* Watchdog flags of a workspace (NULL = this device's internal one); synchronous.
 * Bit 0: a pass-2 block waited more than 4 s for its row's pass-1 result and gave up
 * (a bug: the outputs of that launch are invalid).  reset != 0 clears the flags.
 * Returns -1 on a CUDA error. */
int softmax_watchdog_flags(const void* workspace, int reset);

/* ---- unit-test hooks (device arrays of `count` fp32 values) -----------------
 * what = 0: ExtExp(a) -> (out0 = m, out1 = n)
 *        1: pow2_flush(a) -> out0 = 2^a or 0 (a < -126, -inf, NaN)
 *        2: pair merge (a[2i], a[2i+1]) + (b[2i], b[2i+1]) -> (out0, out1)
 *        3: Exp with reconstruction, argument a <= 0 -> out0 (Alg. 4)
 *        4: the kernels' 2^k for integer k (MUFU.EX2, .ftz) -> out0
 *        5: %globaltimer (ns, uint64) into out0 viewed as uint64[count] (timeline marker)
 *        6: the kernels' ExtExp exactly as pass 1 / pass 2 run it (FFMA2, no clamp):
 *           (out0 = m, out1 = n)
 *        7: the kernels' integer-pipe 2^k: out0 = 2^(d - 127) for d = round(a) <= 254,
 *           +0 for d <= 0 (the scale of Alg. 3's accumulate and pass 2, PAPER.md:161, 168,
 *           flushed below 2^-126 per PAPER.md:252-258)
 *        8: warp value of thread pairs (a[2i], a[2i+1]), i = thread, count a multiple of 32:
 *           per warp w, out0[32 w + 0..3] = (M, N) of the kernels' max-first warp value and
 *           (m, n) of the perfect tree of pair merges over the same 32 pairs in lane order
 *           (reading G8; the two agree outside the sub-2^-126 band) */
int tp_debug_op(int what, const float* a, const float* b, float* out0, float* out1, int64_t count,
                cudaStream_t stream);

/* Compute-only throughput probe (roofline evidence, not part of the method): `ctas` CTAs of
 * 512 threads each run `reps` times over one shared-memory block of 16384 synthetic logits:
 * what = 0 pass 1, 1 pass 2 (no store), 2 both; 3-6 instruction throughput (64 per thread
 * per rep: 3 FFMA2, 4 FFMA2 with an immediate, 5 FFMA, 6 integer add-max + shift); 7 pass 1
 * without the warp tree; 8 pass 2 with its stores, 9 the stores alone, 10 the stores through
 * shared memory and one bulk (TMA) store per block, 11 the stores as 256-bit vectors (8-11: sink
 * needs ctas*16 + ctas*16384 floats).  sink: device, ctas*16 floats (results are
 * meaningless; they keep the work alive).  in_dtype TP_IN_F32 / TP_IN_BF16. */
/* Development: a device buffer of 16 uint64 counters (zeroed by the caller) that later
 * cluster-kernel launches accumulate per-role clock cycles into, summed over CTAs
 * (tools/prof_roles.py documents the slots); NULL switches it off. */
int tp_set_profile_buffer(void* device_counters);

/* STREAM-style HBM baselines beside the softmax passes (measurement only):
 * what = 0 copy y = x (8 B/element), 1 scale y = a x (8), 2 in-place scale x = a x (8),
 * 3 read-only sum (4 B/element; one partial per CTA written to y[0..ctas)), 4 / 5 the read-only
 * sum with 8 / 16 independent 128-bit loads in flight per thread (y not written).  Device pointers,
 * 16-byte aligned, n a multiple of 4; ctas = grid size (0 = 4 per SM).  Asynchronous. */
int tp_stream_baseline(int what, float* x, float* y, int64_t n, float a, int64_t ctas, cudaStream_t stream);

/* Per-pass decomposition (measurement only): runs phase `phase` (0-based; Two-Pass
 * 0..1, Three-Pass 0..2) of `algo` alone over every block of x, on the persistent stream
 * kernel.  A phase > 0 uses the row statistics the workspace holds from the previous FULL call
 * of the same algo, shape and dtype with schedule TP_SCHED_STREAM on the same workspace (it
 * does not wait for them); outputs are then those of the full call's final phase when
 * phase = last.  Phase 0 of Two-Pass writes nothing to y (y may be NULL); the Three-Pass
 * phases 0..1 write nothing either except Reload's phase 1 (y = exp(x - mu)).  Rows must be
 * 16-byte aligned (cols * element size a multiple of 16, aligned base pointers), else TP_EINVAL;
 * workspace as for softmax_ex.  Asynchronous. */
int tp_phase_only(int algo, int in_dtype, int phase, const void* x, float* y, int64_t rows, int64_t cols,
                  void* workspace, size_t workspace_bytes, cudaStream_t stream);

/* HBM read-throughput probe (measurement only): the first floor(bytes / chunk_bytes) chunks of
 * x are read with bulk (TMA) copies into shared memory, CTA c taking chunks c, c + ctas, ...
 * through a ring of `stages` buffers of chunk_bytes (chunk_bytes a multiple of 16, stages <= 32,
 * stages x chunk_bytes <= 227 KB).  x: device, 16-byte aligned; sink: device, ctas floats
 * (meaningless).  Asynchronous; TP_EINVAL on bad arguments. */
int tp_read_probe(const void* x, int64_t bytes, int64_t chunk_bytes, int stages, int64_t ctas, float* sink,
                  cudaStream_t stream);

/* HBM copy-throughput probe (measurement only): y = x over the first floor(bytes / chunk_bytes)
 * chunks with bulk (TMA) copies both ways, CTA c taking chunks c, c + ctas, ... (descending when
 * backward != 0) through a ring of `stages` shared-memory buffers; each chunk is stored straight
 * from its stage.  Limits as tp_read_probe; x, y device, 16-byte aligned, not overlapping.
 * Asynchronous; TP_EINVAL on bad arguments. */
int tp_copy_probe(const void* x, void* y, int64_t bytes, int64_t chunk_bytes, int stages, int64_t ctas, int backward,
                  cudaStream_t stream);

/* Accuracy sweep hook (test/metrology only): for i < count, x = the fp32 whose
 * bit pattern is bits0 + i (the caller keeps bits0 + count - 1 <= 0xffffffff); what = 0:
 * ExtExp -> out0 = m, out1 = n; what = 1: Exp with reconstruction (Alg. 4,
 * PAPER.md:234-249) -> out0.  Device output arrays of count floats. */
int tp_exp_sweep(int what, uint32_t bits0, int64_t count, float* out0, float* out1, cudaStream_t stream);

/* Coefficient-search hook (tools/fit_exp_gpu.py; not part of the method): grades Alg. 4's Exp
 * with the HOST coefficients coeffs[0..4] = c1..c5 against the double exponential on
 * x = as_float(bits0 + i * stride), i < count (normal outputs): *max_ulp_bits (device uint,
 * atomicMax of the float bits; zero it first) and *n_over2 (device uint64, count above 2 ulp). */
int tp_exp_fit(const float* coeffs, uint32_t bits0, int64_t count, int stride, unsigned* max_ulp_bits,
               unsigned long long* n_over2, cudaStream_t stream);

int tp_bench_compute(int what, int in_dtype, int64_t ctas, int reps, float* sink, cudaStream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* TWOPASS_H */
