/*
 * gcnb.h — C ABI of the B200-native row-partitioned GCN training hot path
 * (arXiv 2212.05009; reference package `gcnpart`, /root/reference/pkg/src/gcnpart).
 *
 * Every entry point takes plain device pointers, sizes and a cudaStream_t passed
 * as `void*` (NULL = legacy default stream).  No C++ exceptions cross this
 * boundary: each function returns a status code and leaves a message readable
 * through gcnb_last_error() (thread-local).  Status codes mirror the reference's
 * error classes:
 *   GCNB_OK      0
 *   GCNB_EINVAL  1  -> ValueError   (runtime.py:444-445, 482-486; sparse.py:199-200)
 *   GCNB_ECUDA   2  -> RuntimeError (CUDA launch / memory failure)
 *   GCNB_ECOMM   3  -> CommError    (runtime.py:47-48, 93-108: missing message / timeout)
 *   GCNB_EKEY    4  -> KeyError     (sparse.py:249-254: unowned row)
 *
 * Storage conventions:
 *   * dense row blocks are fp32, row-major, row stride `ld` (floats) with
 *     ld = round_up(d, 4); pad columns are kept at exactly 0.0f;
 *   * CSR operators are int32 row_ptr (n_rows+1), int32 col, fp32 val; the
 *     column space of a rank's operator is [own rows | halo rows], the halo
 *     ordered by sender rank ascending then global id ascending — i.e. the
 *     concatenation of the reference's per-sender positional blocks
 *     (runtime.py:203-230, 254-257), so received rows land in place;
 *   * weights W^k are fp32 [d_{k-1}][ld_k] (column stride padded, pad = 0).
 *
 * Deterministic: every reduction (ΔW partials, loss, allreduce) sums in a fixed
 * order, so reruns are bit-identical (the reference's property, README.md:103-109).
 */
#ifndef GCNB_H
#define GCNB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  GCNB_OK = 0,
  GCNB_EINVAL = 1,
  GCNB_ECUDA = 2,
  GCNB_ECOMM = 3,
  GCNB_EKEY = 4
};

enum { GCNB_ACT_RELU = 0, GCNB_ACT_IDENTITY = 1 };

/* ---- library / diagnostics ------------------------------------------- */
const char* gcnb_last_error(void);
int gcnb_version(void);
/* mbarrier-pipeline watchdog (dense_tc / aggwin): trap after `ms` of a stuck
 * wait; default 60000, 0 = never (env GCNB_WATCHDOG_MS at load). */
int gcnb_set_watchdog_ms(int64_t ms);
/* number of kernels this library has launched in this process (all threads) */
uint64_t gcnb_launch_count(void);
int gcnb_device_count(int* out);

/* ---- memory (device arenas that can be shared with peer processes) ----- */
int gcnb_malloc(void** dptr, size_t bytes);
int gcnb_free(void* dptr);
int gcnb_memset_async(void* dptr, int value, size_t bytes, void* stream);
/* cudaIpcMemHandle_t is 64 bytes */
int gcnb_ipc_get_handle(const void* dptr, uint8_t handle_out[64]);
int gcnb_ipc_open_handle(const uint8_t handle[64], void** dptr_out);
int gcnb_ipc_close_handle(void* dptr);
int gcnb_enable_peer_access(int peer_device);

/* ---- timing events (usable inside CUDA-graph capture: external = 1 records
 * an external event node, so per-kernel spans can be timed on graph replay) */
int gcnb_event_create(void** ev);
int gcnb_event_destroy(void* ev);
int gcnb_event_record(void* ev, void* stream, int32_t external);
int gcnb_event_elapsed_ms(void* ev0, void* ev1, float* ms_out);
/* 1 if `stream` is currently capturing a CUDA graph */
int gcnb_stream_is_capturing(void* stream, int32_t* out);

/* ---- L1 kernels: sparse.py --------------------------------------------- */

/* sparse.spmm (sparse.py:196-207): Y[r] = Σ_j A[r,j]·X[j] for r = rows[i]
 * (rows == NULL: r = i), i < n_rows.  Row i accumulates its nonzeros in CSR
 * (ascending column) order; empty rows produce 0. */
int gcnb_spmm_f32(const int32_t* row_ptr, const int32_t* col, const float* val,
                  const int32_t* rows, int32_t n_rows,
                  const float* x, int32_t ldx, int32_t d,
                  float* y, int32_t ldy, void* stream);

/* Windowed form of gcnb_spmm_f32 for ALL own rows (rows == NULL), the SpMM of
 * runtime._fwd_compute / _bwd_compute (runtime.py:299, 346) over a whole row
 * block.  gcnb_window_csr re-orders each row's nonzeros near-first into int2
 * entries {ring slot | column, value bits} (entries: nnz int2, nnear: n_rows
 * int32) — once per operator, `bt` = window half-width in 128-row tiles, n_own =
 * own rows (halo columns are never near).  gcnb_aggwin_f32 then computes
 * Y[r] = act(Σ A[r,j]·X[j]) with the window rows staged in shared memory by TMA
 * (X rows 0..n_rows-1 are the own rows; far columns may index halo rows).
 * Summation order: near entries then far entries, each in CSR order (fixed).
 * act: GCNB_ACT_RELU / GCNB_ACT_IDENTITY, or -1 for a plain store. */
int gcnb_window_csr(const int32_t* row_ptr, const int32_t* col, const float* val, int32_t n_rows,
                    int32_t n_own, int32_t bt, int32_t* nnear, void* entries, void* stream);
int gcnb_aggwin_applies(int32_t d, int32_t bt, int32_t* out);
/* measurement knob: which passes gcnb_aggwin_f32 runs (1 near, 2 far, 3 both = default) */
int gcnb_set_aggwin_passes(int32_t mask);
int gcnb_aggwin_f32(const int32_t* row_ptr, const int32_t* nnear, const void* entries, int32_t n_rows,
                    int32_t bt, const float* x, int32_t ldx, int32_t d, float* y, int32_t ldy, int32_t act,
                    void* stream);

/* sparse.gather_rows (sparse.py:237-261) and the send-side pack of
 * runtime._fwd_send/_bwd_send (runtime.py:289-294, 336-341), fused with the
 * point-to-point send of SimNetwork.send (runtime.py:85-91):
 * segment s (s < n_seg) copies rows x[idx[seg_ptr[s] .. seg_ptr[s+1])] to
 * dst[s] + i*ld_dst (dst[s] may be a peer-mapped NVLink address).  If
 * flags != NULL, after all rows of the launch are globally visible the kernel
 * atomically increments *flags[s] (system scope, release) for every segment
 * with at least one row — the "message arrived" doorbell used by
 * gcnb_wait_flags.  `counter` is a device int (zero-initialised once) used for
 * the last-block election.  Host arrays dst/flags/seg_ptr have n_seg (+1)
 * entries, n_seg <= GCNB_MAX_PEERS. */
#define GCNB_MAX_PEERS 64
int gcnb_pack_rows_f32(const float* x, int32_t ldx, int32_t d,
                       const int32_t* idx, const int32_t* seg_ptr, int32_t n_seg,
                       float* const* dst, int32_t ld_dst,
                       uint64_t* const* flags, int32_t* counter, void* stream);

/* SimNetwork.recv (runtime.py:93-108) for device transports: block the stream
 * until, for each i < n, flags[srcs[i]] >= ++expected[srcs[i]] (expected is a
 * device array of per-source counters owned by the receiver).  On timeout
 * (timeout_ms) the kernel writes 1 to *err and returns; the host maps a
 * nonzero *err to CommError. */
int gcnb_wait_flags(const uint64_t* flags, const int32_t* srcs_host, int32_t n,
                    uint64_t* expected, int32_t* err, int32_t timeout_ms,
                    void* stream);

/* ---- L6 step functions: runtime.py ------------------------------------- */

/* runtime._fwd_compute (runtime.py:297-306) for the row list `rows`:
 *   w != NULL:  H[r] = act((A[r,:]·X)·W)      (reference order, X is d_in wide)
 *   w == NULL:  H[r] = act(A[r,:]·X)          (X already transformed; d_out == d_in)
 * X is the rank's extended block [own | halo] (row stride ldx), H is written
 * at the own-row positions (row stride ldh).  act: GCNB_ACT_*. */
int gcnb_fwd_layer_f32(const int32_t* row_ptr, const int32_t* col, const float* val,
                       const int32_t* rows, int32_t n_rows,
                       const float* x, int32_t ldx, int32_t d_in,
                       const float* w, int32_t d_out,
                       float* h, int32_t ldh, int32_t act, void* stream);

/* Dense transform Y[r] = act(X[r]·W) for r = rows[i] (rows == NULL: r = i),
 * i < n_rows: the `@ w` of runtime.py:299/304 hoisted before aggregation when
 * d_out < d_in, or the second half of a split aggregate-then-transform layer. */
int gcnb_dense_f32(const float* x, int32_t ldx, const int32_t* rows, int32_t n_rows,
                   int32_t d_in, const float* w, int32_t d_out, float* y, int32_t ldy,
                   int32_t act, void* stream);

/* Dense-transform engine selection (process-wide): 0 = auto (tcgen05 3xTF32
 * for d_in, d_out >= 32, register-blocked SIMT fp32 otherwise), 1 = SIMT fp32
 * everywhere, 2 = tcgen05 wherever the tile fits shared memory.  Both engines
 * meet the 1e-4 fp32 bar; they differ in the last bits. */
int gcnb_set_dense_mode(int32_t mode);
/* ΔW engine for contiguous row blocks: 1 (default) = Hᵀ in tensor memory
 * (k_dw_tc2), 0 = both operands' hi/lo in shared memory (k_dw_tc); A/B knob */
int gcnb_set_dw_mode(int32_t v2);
/* *out = 1 when the tcgen05 engine serves act(X·W) for these widths. */
int gcnb_dense_tc_applies(int32_t d_in, int32_t d_out, int32_t* out);
/* H = relu(X·W) over rows 0..n_rows-1 (tcgen05 engine only) and its sign bits:
 * bit m of bits[r*ld_bits + m/32] = (H[r][m] > 0), i.e. σ'(Z) (gcn.py:101-104)
 * for the backward mask at 1/32 of H's bytes.  ld_bits % 4 == 0. */
int gcnb_dense_bits_f32(const float* x, int32_t ldx, int32_t n_rows, int32_t d_in, const float* w, int32_t d_out,
                        float* y, int32_t ldy, uint32_t* bits, int32_t ld_bits, void* stream);
/* Test/tuning knob: force the (lanes per row, float4 chunks per lane) shape of
 * the aggregation kernel for every width it covers (0, 0 = automatic). */
int gcnb_set_agg_shape(int32_t lpr, int32_t vpl);
/* Test/tuning knob: gathers of the aggregation kernel staged through shared
 * memory with cp.async.cg (0, default), batched in registers (1), or staged
 * with L1-allocating cp.async.ca (2). */
int gcnb_set_agg_gather(int32_t mode);

/* runtime._bwd_compute (runtime.py:344-356) for the row list `rows`:
 *   agg[r]   = A_back[r,:]·G                       (G extended, d_k wide)
 *   G_prev[r] = (agg[r]·W^T) ⊙ act'(H_prev[r])     if g_prev != NULL (k > 1)
 *   ΔW_part  += H_prev[r]^T · agg[r]               per block, deterministic
 * Each launch writes gcnb_bwd_grid(...) partial ΔW blocks of d_prev*ld_k floats
 * to dw_partials; reduce them with gcnb_reduce_partials_f32.  act'(h) is
 * (h > 0) for relu (σ'(z) = (z > 0) = (relu(z) > 0), gcn.py:101-104). */
int gcnb_bwd_grid(int32_t n_rows, int32_t d_prev, int32_t d_k, int32_t with_gprev,
                  int32_t* grid_out);
int gcnb_bwd_layer_f32(const int32_t* row_ptr, const int32_t* col, const float* val,
                       const int32_t* rows, int32_t n_rows,
                       const float* g, int32_t ldg, int32_t d_k,
                       const float* h_prev, int32_t ldhp, int32_t d_prev,
                       const float* w, float* g_prev, int32_t ldgp, int32_t act,
                       float* dw_partials, float* workspace, void* stream);
/* ΔW partials alone: ΔW_part += X[r]^T · A[r] over the row list (no
 * aggregation) — the `h.T @ aggregated` of runtime.py:355 when `aggregated`
 * is already resident.  The runtime uses it for the first layer with
 * X = Â·H^0 (the forward's aggregate) and A = G^1:
 * (Â·H^0)^T·G^1 = H^0^T·(Â^T·G^1), so that layer needs no backward aggregation
 * and no backward halo exchange.  Writes gcnb_bwd_grid(n_rows, d_prev, d_k, 0)
 * partial blocks (d_prev*ld_k floats each) like gcnb_bwd_layer_f32. */
int gcnb_dw_f32(const float* x, int32_t ldx, int32_t d_prev, const float* a, int32_t lda, int32_t d_k,
                const int32_t* rows, int32_t n_rows, float* dw_partials, void* stream);
/* The dense part of gcnb_bwd_layer_f32 from an aggregate already resident in
 * `agg` (rows at own-row positions, e.g. gathered by gcnb_spmm_f32 for the
 * interior and boundary row lists of an overlapped exchange): G_prev and the
 * ΔW partials for the row list, gcnb_bwd_grid(n_rows, d_prev, d_k, g_prev != 0)
 * partial blocks. */
int gcnb_bwd_epilogue_f32(const float* agg, int32_t ldagg, int32_t d_k, const float* h_prev, int32_t ldhp,
                          int32_t d_prev, const float* w, float* g_prev, int32_t ldgp, int32_t act,
                          const uint32_t* hbits, int32_t ld_hbits, const int32_t* rows, int32_t n_rows,
                          float* dw_partials, void* stream);
/* (hbits, optional: sign bits of H_prev as written by gcnb_dense_bits_f32 — the
 * G_prev mask then reads ld_hbits words per row instead of H_prev's floats.) */
/* Measurement knob: 1 = every backward layer uses the split (aggregation +
 * dense epilogue) form when given a workspace, 0 = only large-ΔW layers. */
int gcnb_set_split_all(int32_t on);
/* Engine of the fused aggregate+transform layer (gcnb_fwd_layer_f32 with W):
 * 1 (default) = the aggregation kernel with the narrow transform in its
 * epilogue where the widths allow it, 0 = the tile kernel.  Same sums. */
int gcnb_set_fwd_tf(int32_t on);
/* Row stride (floats) of the optional `workspace` of gcnb_bwd_layer_f32 for
 * these widths, or 0 when the fused single-kernel form is always used.  With a
 * workspace of (own rows) × ld floats, large-ΔW layers run as an aggregation
 * kernel (agg → workspace, full occupancy) plus a dense epilogue kernel;
 * results are identical (same accumulation orders). */
int gcnb_bwd_workspace_ld(int32_t d_prev, int32_t d_k, int32_t* ld_out);

/* out[j] = (accumulate ? out[j] : 0) + Σ_{s < n_slots} partials[s*size + j],
 * summed in a fixed (deterministic) order, j < size, size % 4 == 0.  The
 * partials buffer is scratch: it is folded in place when n_slots > 64. */
int gcnb_reduce_partials_f32(const float* partials, int32_t n_slots, int64_t size,
                             float* out, int32_t accumulate, void* stream);
/* The same reduction with the SGD step of runtime._apply_update
 * (runtime.py:359-360) fused: out = ΔW, then w -= lr·out.  size % 4 == 0. */
int gcnb_reduce_sgd_f32(const float* partials, int32_t n_slots, int64_t size,
                        float* out, int32_t accumulate, float* w, float lr, void* stream);

/* runtime._local_loss_grad (runtime.py:309-333): for every own row r < n_rows,
 * label[r] >= 0 marks a labelled row of class label[r].  For labelled rows:
 * max-shifted log-softmax over the d logits H[r], NLL term, and
 * G[r] = (softmax - onehot) * inv_n_labeled ⊙ act'(H[r]); unlabelled rows get
 * G[r] = 0.  *loss_sum (device double) receives Σ NLL over labelled rows,
 * summed in a fixed order.  `scratch` must hold gcnb_loss_scratch_doubles()
 * doubles. */
int gcnb_loss_scratch_doubles(void);
int gcnb_loss_grad_f32(const float* h, int32_t ldh, int32_t n_rows, int32_t d,
                       const int32_t* label, double inv_n_labeled,
                       float* g, int32_t ldg, int32_t act,
                       double* scratch, double* loss_sum, void* stream);
/* gcnb_loss_grad_f32 with the backward halo pack of the last layer fused into
 * its epilogue (north_star subsystem 2; runtime.py:336-341 + SimNetwork.send):
 * every G row is also stored into the receivers' halo slots the plan assigns
 * to it — map[map_ptr[r] .. map_ptr[r+1]) = {segment s, position}, segment s
 * = receiver halo block dst[s] (row stride ldd floats) — and once all blocks'
 * stores are visible the last block increments flags[s] (system-scope
 * release), exactly as gcnb_pack_rows_f32 would after a separate launch. */
int gcnb_loss_grad_pack_f32(const float* h, int32_t ldh, int32_t n_rows, int32_t d, const int32_t* label,
                            double inv_n_labeled, float* g, int32_t ldg, int32_t act, double* scratch,
                            double* loss_sum, const int32_t* map_ptr, const int32_t* map, float* const* dst,
                            uint64_t* const* flags, int32_t n_seg, int32_t ldd, int32_t* counter, void* stream);

/* A halo pack fused into the epilogue of the kernel that produces the rows
 * (runtime.py:289-294 / 336-341 + SimNetwork.send, without the separate
 * gcnb_pack_rows_f32 launch and its re-read of the rows): own row r, as the
 * kernel stores it, is also stored into every receiver slot
 * map[map_ptr[r] .. map_ptr[r+1]) names ({segment, position} int pairs; slot =
 * dst[segment] + position*ldd floats, a peer-mapped NVLink address), and after
 * all of the launch's stores are visible system-wide the last block
 * increments *flags[s] for every segment, as gcnb_pack_rows_f32 does.
 * map_ptr (n_rows+1) and map live on the device; dst and flags are host arrays
 * of n_seg device pointers (flags may be NULL); counter is a zero-initialised
 * device int that no concurrently running kernel shares.  pack == NULL or
 * n_seg == 0: plain kernel. */
typedef struct gcnb_halo_pack {
  const int32_t* map_ptr;
  const int32_t* map;
  float* const* dst;
  uint64_t* const* flags;
  int32_t n_seg;
  int32_t ldd;
  int32_t* counter;
} gcnb_halo_pack;

/* gcnb_dense_f32 over own rows 0..n_rows-1 (bits != NULL: gcnb_dense_bits_f32)
 * with the produced rows packed into the receivers' halos: the transform of a
 * transform-first layer (T^k = H^{k-1}·W^k, runtime.py:297-306 reordered) or the
 * dense half of a split forward layer (H^k = act(Y·W^k)). */
int gcnb_dense_pack_f32(const float* x, int32_t ldx, int32_t n_rows, int32_t d_in, const float* w, int32_t d_out,
                        float* y, int32_t ldy, int32_t act, uint32_t* bits, int32_t ld_bits,
                        const gcnb_halo_pack* pack, void* stream);
/* gcnb_fwd_layer_f32 (w != NULL) over own rows 0..n_rows-1 with H packed. */
int gcnb_fwd_layer_pack_f32(const int32_t* row_ptr, const int32_t* col, const float* val, int32_t n_rows,
                            const float* x, int32_t ldx, int32_t d_in, const float* w, int32_t d_out, float* h,
                            int32_t ldh, int32_t act, const gcnb_halo_pack* pack, void* stream);
/* gcnb_bwd_layer_f32 over own rows 0..n_rows-1 with G_prev packed (g_prev != NULL). */
int gcnb_bwd_layer_pack_f32(const int32_t* row_ptr, const int32_t* col, const float* val, int32_t n_rows,
                            const float* g, int32_t ldg, int32_t d_k, const float* h_prev, int32_t ldhp,
                            int32_t d_prev, const float* w, float* g_prev, int32_t ldgp, int32_t act,
                            float* dw_partials, float* workspace, const gcnb_halo_pack* pack, void* stream);
/* gcnb_bwd_epilogue_f32 over own rows 0..n_rows-1 with G_prev packed. */
int gcnb_bwd_epilogue_pack_f32(const float* agg, int32_t ldagg, int32_t d_k, const float* h_prev, int32_t ldhp,
                               int32_t d_prev, const float* w, float* g_prev, int32_t ldgp, int32_t act,
                               const uint32_t* hbits, int32_t ld_hbits, int32_t n_rows, float* dw_partials,
                               const gcnb_halo_pack* pack, void* stream);

/* allreduce_sum (runtime.py:147-157): out = bufs[0] + bufs[1] + ... in
 * ascending rank order (bit-identical on every rank).  bufs is a host array of
 * p device pointers (local or peer-mapped). */
int gcnb_sum_buffers_f32(const float* const* bufs, int32_t p, int64_t n,
                         float* out, void* stream);
int gcnb_sum_buffers_f64(const double* const* bufs, int32_t p, int64_t n,
                         double* out, void* stream);

/* Distributed allreduce_sum over NVLink (runtime.py:147-157, 127-133):
 * gcnb_push_f32 copies src (n floats, n % 4 == 0) into n_dst destinations
 * (each rank's slot inside every peer's slot buffer, peer-mapped) and rings
 * *flags[i] (+1, system-scope release) after all stores are visible;
 * gcnb_wait_flags on the receiver then gcnb_sum_slots_f32 sums the p slots
 * in ascending rank order: out[j] = Σ_r slots[r*stride + j] (j < n_f32), and
 * *loss_out = Σ_r (double at slots + r*stride + n_f32) when loss_out != NULL. */
int gcnb_push_f32(const float* src, int64_t n, float* const* dst, uint64_t* const* flags,
                  int32_t n_dst, int32_t* counter, void* stream);
int gcnb_sum_slots_f32(const float* slots, int32_t p, int64_t stride, int64_t n_f32,
                       float* out, double* loss_out, void* stream);
/* Ring n doorbells (+1, system-scope release) after all prior stores of the
 * stream's earlier kernels: with gcnb_wait_flags this is a device-side barrier
 * across processes (the barrier of SimNetwork.allreduce, runtime.py:127-133). */
int gcnb_signal_peers(uint64_t* const* flags, int32_t n, void* stream);

/* runtime._apply_update (runtime.py:359-360): W -= lr·ΔW (n floats). */
int gcnb_sgd_f32(float* w, const float* dw, int64_t n, float lr, void* stream);

/* fp64 → fp32 with column padding: dst[i*ld_dst + j] = (float)src[i*ld_src + j]
 * for j < d, 0 for d <= j < ld_dst (host-prepared inputs uploaded as fp64). */
int gcnb_cast_pad_f64_f32(const double* src, int32_t ld_src, int64_t n_rows,
                          int32_t d, float* dst, int32_t ld_dst, void* stream);

/* ---- setup: device communication plan + rank layout ------
 * gcnb_plan_build = comm.build_comm_plan (comm.py:59-93) for all ranks at once:
 * CSR rp/ci (int64, n rows, square), owner (int32 n), p ranks.  Out: *keys_out
 * = library-allocated sorted distinct keys (consumer << 56 | sender << 49 |
 * column), so block (c, s) = pair_bounds[c*p+s] .. pair_bounds[c*p+s+1] is
 * send[s][c] in ascending column order (and consumer c's blocks, in sender
 * order, are its halo in the reference's positional order); rows_sorted =
 * every rank's rows ascending, rank r's at rank_ptr[r] .. rank_ptr[r+1];
 * localpos[v] = v's position among its owner's rows.  Free keys with
 * gcnb_plan_free.  Synchronises `stream` (setup-time only).
 * gcnb_layout_fill = one rank's block of scatter (runtime.py:203-275): the
 * extended CSR over [own rows | halo] for own rows in `layout_rows` order
 * (halo = keys[halo_k0 .. halo_k0+n_halo)), fp64 values, each row sorted by
 * extended column when sort_rows and n_halo > 0; has_halo_out[i] = row i has a
 * halo column (boundary row).  ext_col_out / val_out hold Σ row lengths. */
int gcnb_plan_build(const int64_t* rp, const int64_t* ci, int64_t n, const int32_t* owner, int32_t p,
                    uint64_t** keys_out, int64_t* n_keys_out, int64_t* pair_bounds, int32_t* rows_sorted,
                    int32_t* rank_ptr, int32_t* localpos, void* stream);
int gcnb_plan_free(void* keys);
int gcnb_layout_fill(const int64_t* rp, const int64_t* ci, const double* val, int64_t n, const int32_t* layout_rows,
                     int32_t n_own, const uint64_t* keys, int64_t halo_k0, int64_t n_halo, int32_t sort_rows,
                     int64_t* row_ptr_out, int32_t* ext_col_out, double* val_out, int32_t* has_halo_out,
                     int32_t* colmap_scratch, void* stream);
/* ---- setup: graph ingest on the device, bit-exact with numpy -
 * gcnb_normalize_f64  = sparse.normalize_adjacency(a, add_self_loops=True)
 *   (sparse.py:167-193); two passes: out_ci == NULL sizes out_rp / *nnz_out;
 * gcnb_transpose_f64  = sparse.transpose_sparse (sparse.py:226-234);
 * gcnb_induced_pattern = models.induced_pattern(a, batch, add_diagonal=False)
 *   (models.py:254-276), batch sorted; two passes like normalize;
 *   pos_scratch: n int64 set to -1 by the caller.  All synchronise `stream`. */
int gcnb_normalize_f64(const int64_t* rp, const int64_t* ci, const double* val, int64_t n, int64_t* out_rp,
                       int64_t* out_ci, double* out_val, int64_t* nnz_out, void* stream);
int gcnb_transpose_f64(const int64_t* rp, const int64_t* ci, const double* val, int64_t n_rows, int64_t n_cols,
                       int64_t* out_rp, int64_t* out_ci, double* out_val, void* stream);
int gcnb_induced_pattern(const int64_t* rp, const int64_t* ci, int64_t n, const int64_t* batch, int64_t B,
                         int64_t* pos_scratch, int64_t* out_rp, int64_t* out_ci, double* out_val, int64_t* nnz_out,
                         void* stream);

/* synchronous device -> host copy (library-allocated buffers) */
int gcnb_copy_d2h(void* dst_host, const void* src_dev, size_t bytes);

#ifdef __cplusplus
}
#endif
#endif /* GCNB_H */
