/* drk.h — C ABI of the B200 distributed-ranges kernel library (libdrk.so).
 *
 * One call = one segment-local operation enqueued on a CUDA stream of one device.
 * Everything is enqueue-only and asynchronous; the caller (the Python runtime, or any
 * other host through ctypes / cffi) owns all memory, streams and synchronisation.
 * Pointers are raw device addresses; `stream` is a cudaStream_t passed as void*.
 * Every entry returns 0 on success, otherwise a cudaError_t value or one of the DRK_E_*
 * codes below; drk_last_error() then describes the failure (thread-local string).
 * Arguments are validated before anything is enqueued ("error before any write",
 * reference runtime.py:324-330, algorithms.py:186-187,476-477).
 *
 * The reference (segrange, pure Python + numpy) has no FFI; each entry point below names
 * the per-segment numpy call site it replaces, so a maintainer can bind it there (see
 * INTEGRATION.md for the ctypes stub a segrange task would call).
 */
#ifndef DRK_H
#define DRK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* element types (numpy dtypes float32, float64, int32, int64) */
enum { DRK_F32 = 0, DRK_F64 = 1, DRK_I32 = 2, DRK_I64 = 3 };
/* unsigned element types: sort / gather / bounds only (the reference's sort bench sorts
 * uint64 splitmix64 keys, bench.py:332-345) */
enum { DRK_U32 = 4, DRK_U64 = 5 };
/* binary operators (reference algorithms.py:47-50: add, multiply, minimum, maximum) */
enum { DRK_ADD = 0, DRK_MUL = 1, DRK_MIN = 2, DRK_MAX = 3 };
/* generator kinds for drk_generate (reference repro.py:21-40) */
enum { DRK_GEN_UNIFORM = 0, DRK_GEN_MOD = 1 };
/* library error codes (disjoint from cudaError_t values, which stay below 1000) */
enum { DRK_E_ARG = 1001, DRK_E_DTYPE = 1002, DRK_E_SCRATCH = 1003, DRK_E_JIT = 1004, DRK_E_COMM = 1005 };

int drk_version(void);
const char* drk_last_error(void);
/* number of CUDA devices visible to this process (0 on a host without a GPU) */
int drk_device_count(int* count);

/* ---- stream plumbing (runtime.py:191-280 allocate/copy/wait_all become stream ops) ---- */
/* cudaMemcpyAsync with cudaMemcpyDefault (host<->device, device<->device, peer over NVLink) */
int drk_memcpy_async(void* dst, const void* src, size_t bytes, int device, void* stream);
int drk_memset_async(void* dst, int value, size_t bytes, int device, void* stream);
/* copy `bytes` (multiple of 8) of device results into mapped pinned host memory with a
 * one-CTA kernel instead of a copy engine, so the per-segment result readback of reduce /
 * scan (algorithms.py:147-149, 256-262) never queues behind bulk downloads on other streams */
int drk_readback(void* host_dst, const void* dev_src, size_t bytes, int device, void* stream);
/* device address of mapped pinned host memory (cudaHostGetDevicePointer): reductions store
 * their per-segment result there directly, so reading it costs one stream sync */
int drk_mapped_ptr(const void* host, void** dev);
/* the wait_all barrier for one locale stream (runtime.py:229-245) */
int drk_stream_synchronize(int device, void* stream);
/* let kernels on `device` load/store memory of `peer` (NVLink P2P through NVSwitch) */
int drk_enable_peer_access(int device, int peer);

/* ---- elementwise (map) kernels -------------------------------------------------------
 * Replace `VectorSegment.store_array(values)` of a materialised view
 * (containers.py:65-67 fed by views.py:164-181 `_apply_elementwise`) and the vectorised
 * `for_each` task (algorithms.py:101-111).  One read of each input, one write. */

/* out[i] = in[i]                      — algorithms.copy aligned path, algorithms.py:493-503 */
int drk_copy(int dtype, void* out, const void* in, int64_t n, int device, void* stream);
/* out[i] = *value                     — DistributedVector(init=v), containers.py:110-113 */
int drk_fill(int dtype, void* out, int64_t n, const void* value, int device, void* stream);
/* out[i] = start + i                  — iota / views.enumerate leaf (no reference analogue) */
int drk_iota(int dtype, void* out, int64_t n, int64_t start, int device, void* stream);
/* out[i] = alpha * in[i]              — STREAM scale */
int drk_scale(int dtype, void* out, const void* in, int64_t n, const void* alpha, int device,
              void* stream);
/* out[i] = a[i] + b[i]                — STREAM add, test_algorithms.py:25-31 */
int drk_add(int dtype, void* out, const void* a, const void* b, int64_t n, int device,
            void* stream);
/* out[i] = b[i] + alpha * c[i]        — bench.stream_triad, bench.py:93-99 (two roundings) */
int drk_triad(int dtype, void* out, const void* b, const void* c, int64_t n, const void* alpha,
              int device, void* stream);
/* out[i] = European call price         — bench.black_scholes_call/prices, bench.py:106-126.
 * The reference's arithmetic operation by operation: for fp32 columns only spot is widened
 * (bench.py:109), so vol, exp(-rT), the drift and strike*discount are fp32 operations (numpy's
 * float32 exp replayed bit for bit) and the log, the normal CDFs and the price fp64, rounded
 * once to dtype.  drk_black_scholes_ex with DRK_BS_FAST is the fast tier: fp32 columns priced
 * in fp32 with SFU approximations (rel <= 1e-5 of the reference; HBM-bound at 2^28 options),
 * fp64 columns in fp64 with fma contraction. */
enum { DRK_BS_FAST = 1 };
int drk_black_scholes(int dtype, void* out, const void* spot, const void* strike,
                      const void* rate, const void* volatility, const void* expiry, int64_t n,
                      int device, void* stream);
int drk_black_scholes_ex(int dtype, int flags, void* out, const void* spot, const void* strike,
                         const void* rate, const void* volatility, const void* expiry, int64_t n,
                         int device, void* stream);
/* Device twin of repro.py:21-40 (splitmix64 window [start, start+n) of `seed`):
 *   DRK_GEN_UNIFORM: out[i] = dtype(a + (b - a) * unit_double)   (a=0,b=1: unit_doubles)
 *   DRK_GEN_MOD:     out[i] = dtype(int64(bits % (uint64)a) + (int64)b)
 * bit-identical to the numpy generator followed by astype(dtype). */
int drk_generate(int dtype, void* out, int64_t n, uint64_t seed, uint64_t start, int kind,
                 double a, double b, int device, void* stream);

/* ---- reductions ------------------------------------------------------------------------
 * Replace `_reduce_task` (algorithms.py:153-162): `op.ufunc.reduce(eval_array())`.
 * The result is written to `result_dev` in the accumulator type drk_acc_dtype(dtype, op)
 * (float32 add/mul -> float64, int32 add/mul -> int64, otherwise dtype).  `scratch` must
 * hold drk_reduce_scratch_bytes() bytes, zero-filled once at allocation; it is left
 * zero-filled again after each call, so one scratch serves every call on one stream.
 * n must be >= 1 (the reference drops empty segments, algorithms.py:61-71). */
size_t drk_reduce_scratch_bytes(void);
int drk_acc_dtype(int dtype, int op);
int drk_reduce(int dtype, int op, const void* x, int64_t n, void* result_dev, void* scratch,
               int device, void* stream);
/* fused zip|transform(t[0]*t[1])|reduce(add) — bench.dot_product, bench.py:87-90 */
int drk_dot(int dtype, const void* x, const void* y, int64_t n, void* result_dev,
            void* scratch, int device, void* stream);

/* ---- scans -----------------------------------------------------------------------------
 * Replace `_local_scan_task` + `_offset_task` / `_seed_task` (algorithms.py:277-308) with a
 * single-pass decoupled look-back scan; the cross-segment carry is an input instead of a
 * second read-modify-write pass.  Values in the accumulator type A = drk_acc_dtype():
 *   init_host     exclusive scans: host pointer to init (A), required; else NULL
 *   carry_host    host pointer to a carry value (A), or NULL
 *   carry_dev     device pointer to a carry value (A) written by an earlier call on the
 *                 same stream (segment chaining), or NULL; at most one carry may be given
 *   seg_total_dev out: this segment's total, without carry (A), or NULL
 *   carry_out_dev out: carry ⊕ segment total (A), or NULL
 * inclusive: out[j] = carry ⊕ in[0..j];  exclusive: out[0] = init ⊕ carry,
 * out[j] = init ⊕ carry ⊕ in[0..j-1].  in == out (in place) is allowed.  n >= 1.
 * `scratch` must hold drk_scan_scratch_bytes(dtype, op, n) bytes, be zero-filled once when
 * allocated, and be used only by drk_scan calls on one stream (tile descriptors are
 * epoch-tagged per call, so nothing is cleared between calls). */
size_t drk_scan_scratch_bytes(int dtype, int op, int64_t n);
int drk_scan(int dtype, int op, int exclusive, const void* in, void* out, int64_t n,
             const void* init_host, const void* carry_host, const void* carry_dev,
             void* seg_total_dev, void* carry_out_dev, void* scratch, size_t scratch_bytes,
             int device, void* stream);

/* Cross-segment scan carry on the device (algorithms.py:256-262, the driver's fold of segment
 * totals): carry_out = carry_in ⊕ L(total_0) ⊕ ... ⊕ L(total_{count-1}) in the accumulator
 * type of drk_acc_dtype(dtype, op), skipping totals whose int64 has-flag is 0 (has may be
 * NULL).  totals / has are arrays of device addresses — peer memory of the GPUs that reduced
 * them, or an all-gathered buffer.  carry_in is a host value (carry_in_host) and/or an earlier
 * fold on the device (carry_in_dev, not re-rounded); either may be NULL.  With nothing to
 * fold the fold's identity is written.  count <= DRK_CARRY_MAX. */
#define DRK_CARRY_MAX 64
int drk_carry_fold(int dtype, int op, const void* const* totals, const void* const* has, int count,
                   const void* carry_in_host, const void* carry_in_dev, void* carry_out_dev, int device,
                   void* stream);

/* drk_scan with flags.  DRK_SCAN_CHAINED: this scan continues a chain of segment scans on
 * one stream — it is launched as a programmatic dependent of the kernel enqueued just before
 * (the scan of the previous segment, which writes this scan's carry_dev).  Its tiles reduce
 * their input while the previous scan drains and wait for it only to read the carry.  The
 * caller guarantees that the previous kernel on the stream is that scan, that the two
 * scans' data do not overlap, and that consecutive scans of a chain use different scratch
 * buffers (alternate two).  Large segments only; otherwise the flag is ignored. */
#define DRK_SCAN_CHAINED 1
int drk_scan_ex(int dtype, int op, int exclusive, int flags, const void* in, void* out, int64_t n,
                const void* init_host, const void* carry_host, const void* carry_dev, void* seg_total_dev,
                void* carry_out_dev, void* scratch, size_t scratch_bytes, int device, void* stream);

/* Scan of a fused view (algorithms.py:198-202 + views.py:164-181 without the temporary):
 * out = scan(f(leaves)) reading only the view's leaves.  `words` (nwords <= 16) describe the
 * view in 8-byte words:
 *   DRK_VIEW_PRODUCT  f = x[i] * y[i]            words {x, y}                (one rounding)
 *   DRK_VIEW_AFFINE   f = alpha * x[i] (+ beta)  words {x, bits(alpha), bits(beta), 1 if beta}
 * (constants as bit patterns in dtype).  vec_ok = every leaf 16-byte aligned; with out also
 * 16-byte aligned and n large the L2 two-touch kernel runs, else the single-pass kernel.
 * op must be DRK_ADD (other operators: NVRTC, drk_jit_scan_view).  Other arguments and the
 * scratch (drk_scan_scratch_bytes) as drk_scan; flags as drk_scan_ex. */
enum { DRK_VIEW_PRODUCT = 1, DRK_VIEW_AFFINE = 2 };
int drk_scan_view(int kind, int dtype, int op, int exclusive, const uint64_t* words, int nwords, int vec_ok,
                  void* out, int64_t n, const void* init_host, const void* carry_host, const void* carry_dev,
                  void* seg_total_dev, void* carry_out_dev, void* scratch, size_t scratch_bytes, int device,
                  void* stream);
int drk_scan_view_ex(int kind, int dtype, int op, int exclusive, int flags, const uint64_t* words, int nwords,
                     int vec_ok, void* out, int64_t n, const void* init_host, const void* carry_host,
                     const void* carry_dev, void* seg_total_dev, void* carry_out_dev, void* scratch,
                     size_t scratch_bytes, int device, void* stream);

/* Batched segment scan: the nseg (<= DRK_SCAN_SEGS) segments of a vector that live on one GPU
 * — ins[k] -> outs[k], ns[k] >= 1 elements, 16-byte aligned — scanned in one launch
 * (algorithms.py:234-308): segment k starts from C_k = carry ⊕ L(T_0) ⊕ .. ⊕ L(T_{k-1}),
 * the segment totals T rounded to numpy's accumulate dtype like the reference's driver fold,
 * passed on the device from the last tile of segment k-1; the first segment starts from
 * carry_host or carry_dev.  seg_totals_dev (nullable) receives each segment's own total in
 * 8-byte slots (accumulator type), carry_out_dev (nullable) C_nseg.  Scratch:
 * drk_scan_batch_scratch_bytes (zeroed once, reusable). */
#define DRK_SCAN_SEGS 16
size_t drk_scan_batch_scratch_bytes(int dtype, int op, int nseg, const int64_t* ns);
int drk_scan_batch(int dtype, int op, int exclusive, int nseg, const void* const* ins, void* const* outs,
                   const int64_t* ns, const void* init_host, const void* carry_host, const void* carry_dev,
                   void* seg_totals_dev, void* carry_out_dev, void* scratch, size_t scratch_bytes, int device,
                   void* stream);

/* Batched reductions (algorithms.py:153-162 `_reduce_task` for every segment a GPU holds, one
 * launch): results receives one 8-byte slot per segment (accumulator type, drk_acc_dtype),
 * scratch is nseg x drk_reduce_scratch_bytes().  nseg <= DRK_RED_SEGS. */
#define DRK_RED_SEGS 16
int drk_reduce_batch(int dtype, int op, int nseg, const void* const* xs, const int64_t* ns, void* results,
                     void* scratch, int device, void* stream);
/* bench.py:87-90 dot_product over every segment pair a GPU holds, one launch */
int drk_dot_batch(int dtype, int nseg, const void* const* xs, const void* const* ys, const int64_t* ns,
                  void* results, void* scratch, int device, void* stream);
/* The batched reductions with completion words: once segment k's result is final (and
 * visible to the host), flags[k] (nullable; nseg 8-byte words, typically mapped pinned host
 * memory beside `results`) is set to `epoch`.  drk_wait_flags spins on the host until every
 * word equals epoch — lower latency than a stream synchronisation for a scalar result; the
 * stream is still checked for errors while waiting. */
int drk_reduce_batch_ex(int dtype, int op, int nseg, const void* const* xs, const int64_t* ns, void* results,
                        void* flags, uint64_t epoch, void* scratch, int device, void* stream);
int drk_dot_batch_ex(int dtype, int nseg, const void* const* xs, const void* const* ys, const int64_t* ns,
                     void* results, void* flags, uint64_t epoch, void* scratch, int device, void* stream);
int drk_wait_flags(const void* host_flags, int count, uint64_t epoch, int device, void* stream);

/* drk_reduce_multi with the cross-GPU combine fused into the kernels (the driver's fold,
 * algorithms.py:146-149, over peer memory): segment k of the listing (device by device, as
 * drk_reduce_multi) stores its partial into home_slots[slot_of[k]] (8-byte accumulator slots
 * on devices[0]; an NVLink peer store from the other GPUs), fences system-wide and takes a
 * ticket on home_counter (4 bytes on devices[0], zero at rest); the CTA with the last ticket
 * folds every slot in order from init (a drk_partial_dtype value) into result_host_mapped,
 * re-arms the counter and sets flag_host_mapped (8 bytes) to epoch — wait with
 * drk_wait_flags(host address of the flag, 1, epoch, ...).  Total segments <= DRK_FOLD_MAX. */
int drk_reduce_fused(int kind, int dtype, int op, int ndev, const int* devices, void* const* streams,
                     const int* counts, const void* const* xs, const void* const* ys, const int64_t* ns,
                     const int* slot_of, void* home_slots, void* home_counter, const void* init,
                     void* result_host_mapped, void* flag_host_mapped, uint64_t epoch, void* const* scratch);

/* One process per GPU: an all-gather of one (has, value) pair per rank over peer memory,
 * without NCCL.  drk_ipc_alloc allocates (and zeroes) a whole device allocation — a rank's
 * mailbox of 2 x world x 32 bytes (two banks, alternating by epoch) — drk_ipc_handle exports
 * it (64-byte cudaIpcMemHandle_t),
 * drk_ipc_open maps another process's on `device` (peer access enabled lazily), drk_ipc_close /
 * drk_ipc_free release them.  drk_mailbox_allgather enqueues one kernel: it stores the rank's
 * 16-byte pair (device memory) into slot `rank` of every mailbox (peer_boxes[j] = rank j's,
 * mapped; the rank's own included), fences system-wide, stamps the slot with epoch, waits
 * until every slot of its own mailbox carries epoch and writes the pairs, rank by rank, into
 * gathered (world x 16 bytes, the layout of an NCCL all-gather).  *status (int, device memory)
 * becomes 0, or 1 when a rank did not arrive within timeout_ns (gathered is then zero there).
 * Epochs must increase from call to call and agree across ranks.  world <= DRK_COMM_MAX_RANKS. */
#define DRK_COMM_MAX_RANKS 32
int drk_ipc_alloc(size_t bytes, int device, void** dev_ptr);
int drk_ipc_free(void* dev_ptr);
int drk_ipc_handle(void* dev_ptr, void* handle_out);
int drk_ipc_open(const void* handle, int device, void** dev_ptr);
int drk_ipc_close(void* dev_ptr);
int drk_mailbox_allgather(const void* pair, void* const* peer_boxes, int world, int rank, const void* own_box,
                          uint64_t epoch, uint64_t timeout_ns, void* gathered, void* status, int device,
                          void* stream);

/* CUDA graphs of fixed launch sequences (a cached plan that issues several kernels on one
 * stream): drk_graph_begin starts a thread-local capture on `stream`, the entries called
 * next are captured instead of run, drk_graph_end instantiates them into *exec (the capture
 * consumed nothing), drk_graph_launch replays them on a stream of the same device,
 * drk_graph_destroy frees *exec.  drk_launch_count counts a replay's kernels. */
int drk_graph_begin(int device, void* stream);
int drk_graph_end(int device, void* stream, void** exec);
int drk_graph_launch(void* exec, int device, void* stream);
int drk_graph_destroy(void* exec);
/* The batched multi-device variant: every GPU's batched reduction (kind 0) or
 * dot (kind 1) of one algorithm call in one entry.  Segments are listed device by device —
 * counts[d] (1..DRK_RED_SEGS) of them on devices[d] / streams[d] — and device d writes its
 * segments' results to results[d] (8-byte slots), its completion words to flags[d] (flags
 * nullable), using scratch[d] (counts[d] x drk_reduce_scratch_bytes()).  Every device's
 * arguments are validated before anything is enqueued. */
int drk_reduce_multi(int kind, int dtype, int op, int ndev, const int* devices, void* const* streams,
                     const int* counts, const void* const* xs, const void* const* ys, const int64_t* ns,
                     void* const* results, void* const* flags, uint64_t epoch, void* const* scratch);

/* ---- cross-GPU combine of a reduce (reference algorithms.py:146-149) ---------------------
 * The driver's ascending fold of per-segment partials, on the device.  partials[k] is the
 * device address (own memory, NVLink peer memory, or an all-gathered buffer) of segment k's
 * partial in the accumulator type (drk_acc_dtype); each is rounded to numpy's reduce dtype
 * P = drk_partial_dtype(dtype, op) (float32 stays float32, int32 sums widen to int64) and
 * folded from init (a P value) in segment order:  r = ((init op P0) op P1) ...
 * The result (a P value) goes to result_dev and/or result_host_mapped (mapped pinned host
 * memory).  count <= DRK_FOLD_MAX. */
#define DRK_FOLD_MAX 64
int drk_partial_dtype(int dtype, int op);
int drk_reduce_fold(int dtype, int op, const void* const* partials, int count, const void* init,
                    void* result_dev, void* result_host_mapped, int device, void* stream);

/* A single-process NCCL communicator over ndev (<= DRK_COMM_MAX_DEV) distinct GPUs
 * (ncclCommInitAll; NCCL is loaded at run time, drk_comm_available() says whether it can be).
 * drk_comm_allgather: GPU i contributes `words` 8-byte words from send[i] and receives
 * ndev * words into recv[i], on streams[i] (one NCCL group).
 * drk_comm_reduce: the whole combine of one reduce in one call — all-gather of every GPU's
 * `words` partial slots (slots[i], padded), then on every GPU the drk_reduce_fold of the
 * gathered partials in segment order (order[k] = gathered word of segment k): every GPU ends
 * with the same result (result_dev[i], array nullable), independent of NCCL's reduction
 * order; GPU 0 also stores it into result_host_mapped (nullable). */
#define DRK_COMM_MAX_DEV 16
int drk_comm_available(void);
int drk_comm_version(void);
int drk_comm_create(int ndev, const int* devices, void** comm);
int drk_comm_destroy(void* comm);
int drk_comm_allgather(void* comm, const void* const* send, void* const* recv, size_t words,
                       void* const* streams);
int drk_comm_reduce(void* comm, int dtype, int op, const void* const* slots, void* const* gather, size_t words,
                    const int* order, int count, const void* init, void* const* result_dev,
                    void* result_host_mapped, void* const* streams);

/* ---- sort (reference algorithms.py:315-432) ------------------------------------------------
 * This library's LSD radix sort (8-bit digits; upsweep / scan / stable downsweep per pass)
 * of one contiguous buffer (a segment, or a sample-sort chunk), n < 2^31, in numpy's order
 * (NaN last), plus the splitter search of the distributed sample sort; the runtime moves
 * the runs between GPUs (peer copies) exactly as the reference's redistribution does.
 * With scratch == NULL, *scratch_bytes receives the required scratch size. */
int drk_sort_keys(int dtype, void* keys, void* alt, int64_t n, void* scratch, size_t* scratch_bytes,
                  int device, void* stream);
/* stable sort of (key, int64 index) pairs by key, in place: keys end sorted, idx permuted alongside */
int drk_sort_pairs(int key_dtype, void* keys, void* keys_alt, void* idx, void* idx_alt, int64_t n,
                   void* scratch, size_t* scratch_bytes, int device, void* stream);
/* out[i] = in[idx[i]] (idx: int64) */
int drk_gather(int dtype, void* out, const void* in, const void* idx, int64_t n, int device, void* stream);
/* sample-sort redistribution bounds (algorithms.py:371-378 `_count_task` on a sorted run):
 * bounds[j] = searchsorted(sorted[0:n], split[j], side="right") in numpy's order (NaN last);
 * split (dtype) and bounds (int64) are device arrays of nsplit entries */
int drk_sort_bounds(int dtype, const void* sorted, int64_t n, const void* split, int nsplit, void* bounds,
                    int device, void* stream);

/* ---- tuning / introspection ------------------------------------------------------------ */
/* set a launch parameter by name ("map_waves", "reduce_waves"); returns the old value */
int drk_tune(const char* name, int value);
/* debug: when non-null, scans record 8 uint64 per tile (%globaltimer stamps: ticket, data
 * ready, aggregate published, look-back done, outputs staged, end; look-back rounds; SM) */
int drk_scan_set_trace(void* buffer);
/* number of kernels this library has launched in this process */
int64_t drk_launch_count(void);

/* ---- run-time compiled kernels (NVRTC) for traced view expressions ----------------------
 * drk_jit_compile compiles CUDA C++ `source` (which may #include "drk_device.cuh" from
 * `include_dir`) for sm_100a and loads it; `*handle` identifies the module.  drk_jit_launch
 * launches `kernel` from that module on (device, stream) with a packed argument block
 * (`params`, `params_bytes`, passed by value as the kernel's single argument). */
int drk_jit_compile(const char* source, const char* name, const char* include_dir,
                    void** handle, char* log, size_t log_bytes);
int drk_jit_cubin(const char* source, const char* name, const char* include_dir,
                  void* cubin_out, size_t* cubin_bytes, char* log, size_t log_bytes);
int drk_jit_load(const void* cubin, void** handle);
int drk_jit_launch(void* handle, const char* kernel, unsigned grid, unsigned block,
                   unsigned smem, const void* params, size_t params_bytes, int device,
                   void* stream);
int drk_jit_occupancy(void* handle, const char* kernel, unsigned block, unsigned smem,
                      int device, int* blocks_per_sm, int* sm_count);

/* scan with an NVRTC-compiled scan kernel (a custom associative operator): the kernel
 * `kernel` of module `handle` must be a scan_kernel instantiation over a plain input with
 * accumulator size acc_bytes (4 or 8), tile = elements per CTA, smem_bytes = its dynamic
 * shared memory.  Other arguments as drk_scan; scratch of drk_jit_scan_scratch_bytes(). */
size_t drk_jit_scan_scratch_bytes(int64_t n, int tile);
int drk_jit_scan(void* handle, const char* kernel, int acc_bytes, int tile, int smem_bytes, int exclusive,
                 const void* in, void* out, int64_t n, const void* init_host, const void* carry_host,
                 const void* carry_dev, void* seg_total_dev, void* carry_out_dev, void* scratch,
                 size_t scratch_bytes, int device, void* stream);
/* scan of a fused view with an NVRTC module that defines drk_scan_l2_s / drk_scan_l2_l (the L2
 * scan over its generated loader with `items` elements per thread and subs_small / subs_large
 * sub-tiles, nl staged leaves — 0 for a register loader) and drk_scan_1p (single pass,
 * items_1p per thread), for values of v_bytes and an accumulator of acc_bytes: other
 * arguments as drk_scan_view_ex; scratch of drk_jit_scan_scratch_bytes(n, 256 * items_1p). */
int drk_jit_scan_view(void* handle, int v_bytes, int acc_bytes, int items, int nl, int subs_small, int subs_large,
                      int items_1p, int exclusive, int flags, const uint64_t* words, int nwords, int vec_ok,
                      void* out, int64_t n, const void* init_host, const void* carry_host, const void* carry_dev,
                      void* seg_total_dev, void* carry_out_dev, void* scratch, size_t scratch_bytes, int device,
                      void* stream);
const char* drk_jit_last_error(void);
int64_t drk_note_launch(void);

#ifdef __cplusplus
}
#endif
#endif /* DRK_H */
