// drk_scan.cu — launchers of the scan kernels (drk_device.cuh): single segments (plain and
// fused views), batched segments, and the C ABI entries drk_scan*, drk_scan_batch*,
// drk_scan_view*, drk_jit_scan_view (include/drk.h).  Split from drk_kernels.cu so the
// library's template instantiations compile in parallel.
#include "drk_host.h"

using namespace drk;
using namespace drk_host;

// ---------------------------------------------------------------------------------------
// scans

// Launch an L2-scan kernel (AOT template instance or NVRTC kernel, given as a function
// pointer) over ntiles tiles: stagger and early-trigger policy, and the programmatic-
// dependent launch of a chained segment scan (drk_scan_ex DRK_SCAN_CHAINED).
template <class A, class LP>
static int launch_l2_fn(const void* fn, ScanParams<A, LP>& p, int64_t tile, int smem, int device, cudaStream_t s,
                        bool two_phase = false) {
  const int64_t nt = (p.n + tile - 1) / tile;
  if (nt > 0x7fffffffLL) return set_error(DRK_E_ARG, "drk_scan: too many tiles");
  p.ntiles = (u32)nt;
  smem += g_scan_smem_pad;
  p.rescan_pol = g_scan_rescan_pol;
  p.keep_tail = g_scan_keep_tail;
  p.lb_snap = g_scan_lb_snap;
  DRK_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  // With more than two waves of tiles, every CTA lets a chained successor launch as soon as
  // it starts (a no-op unless the next kernel is a DRK_SCAN_CHAINED scan): all of this grid
  // has started only after most of it has finished, i.e. after its own wait for the scan
  // before it, whose scratch the successor reuses.
  const int64_t wave = (int64_t)sm_count(device) * occupancy(fn, BLOCK, smem);
  p.early_trigger = nt > 2 * wave;
  // Stagger the first wave's reduces (ticket order) when the grid spans several waves:
  // 2^26-2^28 elements gain 4-6 %; a single wave gains nothing (all tiles must be read
  // before the last look-back resolves anyway)
  p.stagger_tiles = (u32)wave;
  if (g_scan_stagger < 0) p.stagger_ns = nt > 2 * wave ? 40 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)nt);
  cfg.blockDim = dim3(BLOCK);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  if (g_chain_launch) {
    // programmatic dependent of the previous scan of the chain (see carry_dev_read)
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  void* args[] = {&p};
  if (two_phase && !g_chain_launch) {
    // every tile reduces and publishes its aggregate, then a second launch over the same
    // tiles (same epoch) scans them from L2 with every aggregate already published
    p.stagger_ns = 0;
    p.early_trigger = 0;
    p.phase = 1;
    DRK_CHECK(cudaLaunchKernelExC(&cfg, fn, args));
    drk_note_launch();  // the second launch is counted by the caller's epilogue
    p.phase = 2;
  }
  DRK_CHECK(cudaLaunchKernelExC(&cfg, fn, args));
  return 0;
}

// 160 KB tiles (8 x 20 KB for 4-byte types); below 2^25 elements (about one wave of tiles)
// 80 KB tiles, which give the grid more waves (2^23: 32.8 -> 26.9 us).  Other tile sizes
// measured (3, 6, 7, 10, 12 sub-tiles) are not instantiated.
static int l2_subs(int64_t n) { return g_scan_l2_subs == 4 || g_scan_l2_subs == 8 ? g_scan_l2_subs
                                                                                   : (n < ((int64_t)1 << 25) ? 4 : 8); }

template <class LDR, class Op>
static int launch_scan_l2_any(ScanParams<typename WideAcc<typename LDR::V, Op>::type, typename LDR::Params>& p,
                              int device, cudaStream_t s) {
  typedef typename LDR::V T;
  constexpr int IT = ScanItems<T, Op>::value;
  const int subs = l2_subs(p.n);
  p.pre = g_scan_l2_pre;
  const int smem = 3 * BLOCK * IT * (int)sizeof(T);
  const void* fn = subs == 4 ? (const void*)scan_l2_kernel<LDR, Op, BLOCK, IT, 4, 3>
                             : (const void*)scan_l2_kernel<LDR, Op, BLOCK, IT, 8, 3>;
  const int64_t in_kb = p.n * (int64_t)sizeof(T) * (LDR::NL > 1 ? LDR::NL : 1) >> 10;
  const bool two = p.nseg == 0 && g_scan_2p_hi_kb > 0 && in_kb >= g_scan_2p_lo_kb && in_kb <= g_scan_2p_hi_kb;
  return launch_l2_fn(fn, p, (int64_t)BLOCK * IT * subs, smem, device, s, two);
}

template <class T, class Op, int SUB>
static int launch_scan_sub(ScanParams<typename WideAcc<T, Op>::type, const T*>& p, int64_t n, int device,
                           cudaStream_t s) {
  constexpr int ITEMS = ScanItems<T, Op>::value;
  typedef ScanConfig<T, T, Op, BLOCK, ITEMS, SUB> C;
  if (p.bulk_ok && g_scan_l2dyn && n >= (int64_t)g_scan_l2_min) return launch_scan_l2_any<PlainLoad<T>, Op>(p, device, s);
  const int64_t nt64 = (n + C::TILE - 1) / C::TILE;
  if (nt64 > 0x7fffffffLL) return set_error(DRK_E_ARG, "drk_scan: too many tiles");
  p.ntiles = (u32)nt64;
  auto k = scan_kernel<PlainLoad<T>, T, Op, BLOCK, ITEMS, SUB>;
  if (C::SMEM > 48 * 1024) DRK_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  k<<<p.ntiles, BLOCK, C::SMEM, s>>>(p);
  return 0;
}

template <class T, class Op>
static int launch_scan(int exclusive, const T* in, T* out, int64_t n, const void* init_host, const void* carry_host,
                       const void* carry_dev, void* seg_total, void* carry_out, void* scratch, size_t scratch_bytes,
                       int device, void* stream) {
  typedef typename WideAcc<T, Op>::type A;
  const char* what = "drk_scan";
  if (n < 1) return set_error(DRK_E_ARG, "drk_scan: n must be >= 1");
  if (!in || !out) return set_error(DRK_E_ARG, "drk_scan: null in/out");
  if (exclusive && !init_host) return set_error(DRK_E_ARG, "drk_scan: exclusive scan needs init");
  if (carry_host && carry_dev) return set_error(DRK_E_ARG, "drk_scan: give at most one carry");
  const size_t need_bytes = scan_scratch<T, Op>(n);
  if (!scratch || scratch_bytes < need_bytes)
    return set_error(DRK_E_SCRATCH, "drk_scan: scratch too small (need " + std::to_string(need_bytes) + ")");
  if (int rc = prologue(device, what)) return rc;
  char* b = (char*)scratch;
  ScanParams<A, const T*> p;
  memset(&p, 0, sizeof(p));
  p.in = in;
  p.out = out;
  p.n = n;
  p.exclusive = exclusive;
  p.has_init = init_host != nullptr;
  if (init_host) memcpy(&p.init, init_host, sizeof(A));
  p.carry_kind = carry_host ? 1 : (carry_dev ? 2 : 0);
  if (carry_host) memcpy(&p.carry_val, carry_host, sizeof(A));
  p.carry_ptr = (const A*)carry_dev;
  p.seg_total = (A*)seg_total;
  p.carry_out = (A*)carry_out;
  p.counter = (u32*)b;
  p.desc = (u64*)(b + 128);
  p.t0slot = (u64*)(b + 64);
  p.stagger_ns = g_scan_stagger > 0 ? (u32)g_scan_stagger : 0;  // < 0: automatic (launch_l2_fn)
  p.epoch = next_epoch(scratch);
  p.bulk_ok = aligned16(in) && aligned16(out);
  p.trace = (u64*)g_scan_trace;
  p.debug = g_scan_debug;
  cudaStream_t s = (cudaStream_t)stream;
  int rc = 0;
  // sub-tiles per tile of the single-pass kernel (small or unaligned segments): 0 = by size —
  // one 20 KB sub-tile below 2^20 elements (more, shorter-lived tiles: 2^18-2^19 fp32
  // 14.8 -> 10.8 us), two up to 2^21, three above
  const int sub = g_scan_sub > 0 ? g_scan_sub : (n < ((int64_t)1 << 20) ? 1 : (n < ((int64_t)1 << 22) ? 2 : 3));
  switch (sub) {
    case 1: rc = launch_scan_sub<T, Op, 1>(p, n, device, s); break;
    case 3: rc = launch_scan_sub<T, Op, 3>(p, n, device, s); break;
    case 4: rc = launch_scan_sub<T, Op, 4>(p, n, device, s); break;
    default: rc = launch_scan_sub<T, Op, 2>(p, n, device, s); break;
  }
  if (rc) return rc;
  return epilogue(what);
}

template <class T>
static int scan_op(int op, int exclusive, const T* in, T* out, int64_t n, const void* init_host,
                   const void* carry_host, const void* carry_dev, void* seg_total, void* carry_out, void* scratch,
                   size_t sb, int device, void* stream) {
  switch (op) {
    case DRK_ADD:
      return launch_scan<T, OpAdd>(exclusive, in, out, n, init_host, carry_host, carry_dev, seg_total, carry_out,
                                   scratch, sb, device, stream);
    case DRK_MUL:
      return launch_scan<T, OpMul>(exclusive, in, out, n, init_host, carry_host, carry_dev, seg_total, carry_out,
                                   scratch, sb, device, stream);
    case DRK_MIN:
      return launch_scan<T, OpMin>(exclusive, in, out, n, init_host, carry_host, carry_dev, seg_total, carry_out,
                                   scratch, sb, device, stream);
    case DRK_MAX:
      return launch_scan<T, OpMax>(exclusive, in, out, n, init_host, carry_host, carry_dev, seg_total, carry_out,
                                   scratch, sb, device, stream);
  }
  return set_error(DRK_E_ARG, "drk_scan: unknown op");
}

extern "C" size_t drk_scan_scratch_bytes(int dtype, int op, int64_t n) {
  if (n < 1) n = 1;
#define DRK_SS(T)                                               \
  switch (op) {                                                 \
    case DRK_ADD: return scan_scratch<T, OpAdd>(n);             \
    case DRK_MUL: return scan_scratch<T, OpMul>(n);             \
    case DRK_MIN: return scan_scratch<T, OpMin>(n);             \
    case DRK_MAX: return scan_scratch<T, OpMax>(n);             \
    default: return 0;                                          \
  }
  switch (dtype) {
    case DRK_F32: DRK_SS(float)
    case DRK_F64: DRK_SS(double)
    case DRK_I32: DRK_SS(int)
    case DRK_I64: DRK_SS(long long)
  }
#undef DRK_SS
  return 0;
}

extern "C" int drk_scan(int dtype, int op, int exclusive, const void* in, void* out, int64_t n,
                        const void* init_host, const void* carry_host, const void* carry_dev, void* seg_total_dev,
                        void* carry_out_dev, void* scratch, size_t scratch_bytes, int device, void* stream) {
  DRK_DISPATCH(dtype, "drk_scan", T, {
    return scan_op<T>(op, exclusive, (const T*)in, (T*)out, n, init_host, carry_host, carry_dev, seg_total_dev,
                      carry_out_dev, scratch, scratch_bytes, device, stream);
  });
}

// ---------------------------------------------------------------------------------------
// batched segments: one L2-scan launch over up to DRK_SCAN_SEGS buffers on one GPU (the
// segments of a vector that share a device), so there is one ramp-up and one tail instead of
// one per segment.  Each segment's look-back stays inside the segment; its carry comes from
// the last tile of the segment before it (segdesc), as the driver's fold of the rounded
// partials (algorithms.py:234-274), and its total is written straight to seg_totals[k].

static size_t batch_tiles(int dtype, int nseg, const int64_t* ns) {
  const int64_t tile = (int64_t)BLOCK * 8 * ((dtype == DRK_F64 || dtype == DRK_I64) ? 10 : 20);
  size_t nt = 0;
  for (int k = 0; k < nseg; ++k) nt += (size_t)((ns[k] + tile - 1) / tile);
  return nt;
}

extern "C" size_t drk_scan_batch_scratch_bytes(int dtype, int op, int nseg, const int64_t* ns) {
  (void)op;
  return 128 + batch_tiles(dtype, nseg, ns) * 16 + (DRK_SCAN_SEGS + 1) * 16;
}

template <class T, class Op>
static int launch_scan_batch(int exclusive, int nseg, const void* const* ins, void* const* outs, const int64_t* ns,
                             const void* init_host, const void* carry_host, const void* carry_dev, void* seg_totals,
                             void* carry_out, void* scratch, size_t scratch_bytes, int device, void* stream) {
  typedef typename WideAcc<T, Op>::type A;
  constexpr int IT = ScanItems<T, Op>::value;
  constexpr int SUBS = 8;
  constexpr int TILE = BLOCK * IT * SUBS;
  const char* what = "drk_scan_batch";
  if (nseg < 1 || nseg > DRK_SCAN_SEGS) return set_error(DRK_E_ARG, "drk_scan_batch: nseg out of range");
  if (exclusive && !init_host) return set_error(DRK_E_ARG, "drk_scan_batch: exclusive scan needs init");
  if (carry_host && carry_dev) return set_error(DRK_E_ARG, "drk_scan_batch: give at most one carry");
  ScanParams<A, const T*> p;
  memset(&p, 0, sizeof(p));
  u64 nt = 0;
  for (int k = 0; k < nseg; ++k) {
    if (ns[k] < 1 || !ins[k] || !outs[k]) return set_error(DRK_E_ARG, "drk_scan_batch: empty or null segment");
    if (!aligned16(ins[k]) || !aligned16(outs[k]))
      return set_error(DRK_E_ARG, "drk_scan_batch: segments must be 16-byte aligned");
    p.seg_first[k] = (u32)nt;
    p.seg_in[k] = ins[k];
    p.seg_out[k] = outs[k];
    p.seg_n[k] = ns[k];
    nt += (u64)((ns[k] + TILE - 1) / TILE);
  }
  p.seg_first[nseg] = (u32)nt;
  if (nt > 0x7fffffffull) return set_error(DRK_E_ARG, "drk_scan_batch: too many tiles");
  const size_t need = 128 + nt * 16 + (DRK_SCAN_SEGS + 1) * 16;
  if (!scratch || scratch_bytes < need)
    return set_error(DRK_E_SCRATCH, "drk_scan_batch: scratch too small (need " + std::to_string(need) + ")");
  if (int rc = prologue(device, what)) return rc;
  char* b = (char*)scratch;
  p.nseg = nseg;
  p.n = (int64_t)nt * TILE;  // tile count for the launcher (segments carry their own lengths)
  p.exclusive = exclusive;
  p.has_init = init_host != nullptr;
  if (init_host) memcpy(&p.init, init_host, sizeof(A));
  p.carry_kind = carry_host ? 1 : (carry_dev ? 2 : 0);
  if (carry_host) memcpy(&p.carry_val, carry_host, sizeof(A));
  p.carry_ptr = (const A*)carry_dev;
  p.seg_total = (A*)seg_totals;
  p.carry_out = (A*)carry_out;
  p.counter = (u32*)b;
  p.desc = (u64*)(b + 128);
  p.segdesc = (u64*)(b + 128 + nt * 16);
  p.t0slot = (u64*)(b + 64);
  p.epoch = next_epoch(scratch);
  p.bulk_ok = 1;
  p.pre = g_scan_l2_pre;
  p.debug = g_scan_debug;
  p.stagger_ns = g_scan_stagger > 0 ? (u32)g_scan_stagger : 0;
  const int smem = 3 * BLOCK * IT * (int)sizeof(T);
  if (int rc = launch_l2_fn((const void*)scan_l2_kernel<PlainLoad<T>, Op, BLOCK, IT, SUBS, 3>, p, TILE, smem, device,
                            (cudaStream_t)stream))
    return rc;
  return epilogue(what);
}

template <class T>
static int scan_batch_op(int op, int exclusive, int nseg, const void* const* ins, void* const* outs, const int64_t* ns,
                         const void* init_host, const void* carry_host, const void* carry_dev, void* seg_totals,
                         void* carry_out, void* scratch, size_t sb, int device, void* stream) {
  switch (op) {
    case DRK_ADD:
      return launch_scan_batch<T, OpAdd>(exclusive, nseg, ins, outs, ns, init_host, carry_host, carry_dev, seg_totals,
                                         carry_out, scratch, sb, device, stream);
    case DRK_MUL:
      return launch_scan_batch<T, OpMul>(exclusive, nseg, ins, outs, ns, init_host, carry_host, carry_dev, seg_totals,
                                         carry_out, scratch, sb, device, stream);
    case DRK_MIN:
      return launch_scan_batch<T, OpMin>(exclusive, nseg, ins, outs, ns, init_host, carry_host, carry_dev, seg_totals,
                                         carry_out, scratch, sb, device, stream);
    case DRK_MAX:
      return launch_scan_batch<T, OpMax>(exclusive, nseg, ins, outs, ns, init_host, carry_host, carry_dev, seg_totals,
                                         carry_out, scratch, sb, device, stream);
  }
  return set_error(DRK_E_ARG, "drk_scan_batch: unknown op");
}

extern "C" int drk_scan_batch(int dtype, int op, int exclusive, int nseg, const void* const* ins, void* const* outs,
                              const int64_t* ns, const void* init_host, const void* carry_host, const void* carry_dev,
                              void* seg_totals_dev, void* carry_out_dev, void* scratch, size_t scratch_bytes,
                              int device, void* stream) {
  if (!ins || !outs || !ns) return set_error(DRK_E_ARG, "drk_scan_batch: null segment arrays");
  DRK_DISPATCH(dtype, "drk_scan_batch", T, {
    return scan_batch_op<T>(op, exclusive, nseg, ins, outs, ns, init_host, carry_host, carry_dev, seg_totals_dev,
                            carry_out_dev, scratch, scratch_bytes, device, stream);
  });
}

extern "C" int drk_scan_ex(int dtype, int op, int exclusive, int flags, const void* in, void* out, int64_t n,
                           const void* init_host, const void* carry_host, const void* carry_dev,
                           void* seg_total_dev, void* carry_out_dev, void* scratch, size_t scratch_bytes, int device,
                           void* stream) {
  if (flags & ~DRK_SCAN_CHAINED) return set_error(DRK_E_ARG, "drk_scan_ex: unknown flags");
  if ((flags & DRK_SCAN_CHAINED) && !carry_dev)
    return set_error(DRK_E_ARG, "drk_scan_ex: a chained scan takes its carry from the previous scan (carry_dev)");
  g_chain_launch = (flags & DRK_SCAN_CHAINED) != 0;
  const int rc = drk_scan(dtype, op, exclusive, in, out, n, init_host, carry_host, carry_dev, seg_total_dev,
                          carry_out_dev, scratch, scratch_bytes, device, stream);
  g_chain_launch = 0;
  return rc;
}

// ---------------------------------------------------------------------------------------
// scans of fused views: inclusive_scan(transform(x, f), out) reads the leaves of the view and
// writes only `out` (reference views.py:164-181 materialises f(x) first, algorithms.py:198-202
// then scans it).  The loader (AOT ProdScanLoad / AffineScanLoad, or NVRTC-generated) gets
// its leaf pointers and constants as JitWords.

template <class A>
static int fill_view_params(ScanParams<A, JitWords>& p, const uint64_t* words, int nwords, void* out, int64_t n,
                            int exclusive, const void* init_host, const void* carry_host, const void* carry_dev,
                            void* seg_total, void* carry_out, void* scratch, size_t scratch_bytes, size_t need,
                            const char* what) {
  if (n < 1) return set_error(DRK_E_ARG, std::string(what) + ": n must be >= 1");
  if (!out || !words) return set_error(DRK_E_ARG, std::string(what) + ": null out/words");
  if (nwords < 0 || nwords > DRK_JIT_WORDS)
    return set_error(DRK_E_ARG, std::string(what) + ": at most " + std::to_string(DRK_JIT_WORDS) + " words");
  if (exclusive && !init_host) return set_error(DRK_E_ARG, std::string(what) + ": exclusive scan needs init");
  if (carry_host && carry_dev) return set_error(DRK_E_ARG, std::string(what) + ": give at most one carry");
  if (!scratch || scratch_bytes < need)
    return set_error(DRK_E_SCRATCH, std::string(what) + ": scratch too small (need " + std::to_string(need) + ")");
  memset(&p, 0, sizeof(p));
  memcpy(p.in.w, words, sizeof(uint64_t) * nwords);
  p.out = out;
  p.n = n;
  p.exclusive = exclusive;
  p.has_init = init_host != nullptr;
  if (init_host) memcpy(&p.init, init_host, sizeof(A));
  p.carry_kind = carry_host ? 1 : (carry_dev ? 2 : 0);
  if (carry_host) memcpy(&p.carry_val, carry_host, sizeof(A));
  p.carry_ptr = (const A*)carry_dev;
  p.seg_total = (A*)seg_total;
  p.carry_out = (A*)carry_out;
  char* b = (char*)scratch;
  p.counter = (u32*)b;
  p.t0slot = (u64*)(b + 64);
  p.desc = (u64*)(b + 128);
  p.epoch = next_epoch(scratch);
  p.stagger_ns = g_scan_stagger > 0 ? (u32)g_scan_stagger : 0;
  p.trace = (u64*)g_scan_trace;
  p.debug = g_scan_debug;
  return 0;
}

// The kernels of one fused-view scan: the L2 kernel for small (< 2^25) and large inputs and
// the single-pass kernel, with the L2 geometry of the loader (ScanGeom: elements per thread
// and sub-tiles, leaf buffers per ring slot).
struct ViewKernels {
  const void* l2_small;
  const void* l2_large;
  const void* one;
  int v_bytes, items, nlb, subs_small, subs_large, items_1p;
};

// One fused-view scan: the L2 kernel when every leaf is 16-byte aligned (vec_ok), out is too
// and n is large; else the single-pass kernel (3 sub-tiles).
template <class A>
static int launch_view_scan(const ViewKernels& k, ScanParams<A, JitWords>& p, int vec_ok, int device,
                            cudaStream_t s) {
  if (vec_ok && aligned16(p.out) && g_scan_l2dyn && p.n >= (int64_t)g_scan_l2_min) {
    p.bulk_ok = 1;
    p.pre = g_scan_l2_pre;
    const bool small = p.n < ((int64_t)1 << 25);
    const int subs = small ? k.subs_small : k.subs_large;
    return launch_l2_fn(small ? k.l2_small : k.l2_large, p, (int64_t)BLOCK * k.items * subs,
                        3 * k.nlb * BLOCK * k.items * k.v_bytes, device, s);
  }
  constexpr int SUB = 3;
  const int64_t tile = (int64_t)BLOCK * k.items_1p * SUB;
  const int64_t nt = (p.n + tile - 1) / tile;
  if (nt > 0x7fffffffLL) return set_error(DRK_E_ARG, "drk_scan_view: too many tiles");
  p.ntiles = (u32)nt;
  p.bulk_ok = 0;
  const int smem = (int)tile * k.v_bytes;
  DRK_CHECK(cudaFuncSetAttribute(k.one, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)nt);
  cfg.blockDim = dim3(BLOCK);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  void* args[] = {&p};
  DRK_CHECK(cudaLaunchKernelExC(&cfg, k.one, args));
  return 0;
}

template <class LDR, class Op>
static int view_scan_aot(const uint64_t* words, int nwords, int vec_ok, int exclusive, void* out, int64_t n,
                         const void* init_host, const void* carry_host, const void* carry_dev, void* seg_total,
                         void* carry_out, void* scratch, size_t scratch_bytes, int device, void* stream) {
  typedef typename LDR::V T;
  typedef typename WideAcc<T, Op>::type A;
  typedef ScanGeom<(int)sizeof(T), LDR::NL> G;
  constexpr int IT1 = ScanItems<T, Op>::value;
  const char* what = "drk_scan_view";
  ScanParams<A, JitWords> p;
  if (int rc = fill_view_params(p, words, nwords, out, n, exclusive, init_host, carry_host, carry_dev, seg_total,
                                carry_out, scratch, scratch_bytes, scan_scratch<T, Op>(n), what))
    return rc;
  if (int rc = prologue(device, what)) return rc;
  const ViewKernels k = {(const void*)scan_l2_kernel<LDR, Op, BLOCK, G::ITEMS, G::SUBS_SMALL, 3>,
                         (const void*)scan_l2_kernel<LDR, Op, BLOCK, G::ITEMS, G::SUBS_LARGE, 3>,
                         (const void*)scan_kernel<LDR, T, Op, BLOCK, IT1, 3>,
                         (int)sizeof(T), G::ITEMS, LDR::NL > 0 ? LDR::NL : 1, G::SUBS_SMALL, G::SUBS_LARGE, IT1};
  if (int rc = launch_view_scan(k, p, vec_ok, device, (cudaStream_t)stream)) return rc;
  return epilogue(what);
}

extern "C" int drk_scan_view(int kind, int dtype, int op, int exclusive, const uint64_t* words, int nwords,
                             int vec_ok, void* out, int64_t n, const void* init_host, const void* carry_host,
                             const void* carry_dev, void* seg_total_dev, void* carry_out_dev, void* scratch,
                             size_t scratch_bytes, int device, void* stream) {
  if (op != DRK_ADD) return set_error(DRK_E_ARG, "drk_scan_view: the AOT view scans take op = DRK_ADD");
  if (kind != DRK_VIEW_PRODUCT && kind != DRK_VIEW_AFFINE) return set_error(DRK_E_ARG, "drk_scan_view: unknown kind");
  DRK_DISPATCH(dtype, "drk_scan_view", T, {
    if (kind == DRK_VIEW_PRODUCT)
      return view_scan_aot<ProdScanLoad<T>, OpAdd>(words, nwords, vec_ok, exclusive, out, n, init_host, carry_host,
                                                    carry_dev, seg_total_dev, carry_out_dev, scratch, scratch_bytes,
                                                    device, stream);
    return view_scan_aot<AffineScanLoad<T>, OpAdd>(words, nwords, vec_ok, exclusive, out, n, init_host, carry_host,
                                                    carry_dev, seg_total_dev, carry_out_dev, scratch, scratch_bytes,
                                                    device, stream);
  });
}

extern "C" int drk_scan_view_ex(int kind, int dtype, int op, int exclusive, int flags, const uint64_t* words,
                                int nwords, int vec_ok, void* out, int64_t n, const void* init_host,
                                const void* carry_host, const void* carry_dev, void* seg_total_dev,
                                void* carry_out_dev, void* scratch, size_t scratch_bytes, int device, void* stream) {
  if (flags & ~DRK_SCAN_CHAINED) return set_error(DRK_E_ARG, "drk_scan_view_ex: unknown flags");
  if ((flags & DRK_SCAN_CHAINED) && !carry_dev)
    return set_error(DRK_E_ARG, "drk_scan_view_ex: a chained scan takes its carry from the previous scan");
  g_chain_launch = (flags & DRK_SCAN_CHAINED) != 0;
  const int rc = drk_scan_view(kind, dtype, op, exclusive, words, nwords, vec_ok, out, n, init_host, carry_host,
                               carry_dev, seg_total_dev, carry_out_dev, scratch, scratch_bytes, device, stream);
  g_chain_launch = 0;
  return rc;
}

// NVRTC view scans: the module defines drk_scan_l2_s / drk_scan_l2_l (scan_l2_body with
// `items` elements per thread and subs_small / subs_large sub-tiles, nl staged leaves or 0
// for a register loader) and drk_scan_1p (scan_kernel_body, items_1p, 3 sub-tiles).
extern "C" int drk_get_jit_kernel(void* handle, const char* kernel, const void** fn);

extern "C" int drk_jit_scan_view(void* handle, int v_bytes, int acc_bytes, int items, int nl, int subs_small,
                                 int subs_large, int items_1p, int exclusive, int flags, const uint64_t* words,
                                 int nwords, int vec_ok, void* out, int64_t n, const void* init_host,
                                 const void* carry_host, const void* carry_dev, void* seg_total_dev,
                                 void* carry_out_dev, void* scratch, size_t scratch_bytes, int device, void* stream) {
  const char* what = "drk_jit_scan_view";
  if (v_bytes != 4 && v_bytes != 8) return set_error(DRK_E_ARG, "drk_jit_scan_view: v_bytes must be 4 or 8");
  if (items < 1 || items_1p < 1 || subs_small < 1 || subs_large < 1 || nl < 0 || nl > 4)
    return set_error(DRK_E_ARG, "drk_jit_scan_view: bad geometry");
  if (flags & ~DRK_SCAN_CHAINED) return set_error(DRK_E_ARG, "drk_jit_scan_view: unknown flags");
  ViewKernels k = {nullptr, nullptr, nullptr, v_bytes, items, nl > 0 ? nl : 1, subs_small, subs_large, items_1p};
  if (int rc = drk_get_jit_kernel(handle, "drk_scan_l2_s", &k.l2_small)) return set_error(rc, "drk_jit_scan_view: no kernel");
  if (int rc = drk_get_jit_kernel(handle, "drk_scan_l2_l", &k.l2_large)) return set_error(rc, "drk_jit_scan_view: no kernel");
  if (int rc = drk_get_jit_kernel(handle, "drk_scan_1p", &k.one)) return set_error(rc, "drk_jit_scan_view: no kernel");
  const int64_t t1 = (int64_t)BLOCK * items_1p;
  const size_t need = 128 + (size_t)((n + t1 - 1) / t1) * 16;
  if (int rc = prologue(device, what)) return rc;
  g_chain_launch = (flags & DRK_SCAN_CHAINED) != 0;
  int rc = 0;
  if (acc_bytes == 8) {
    ScanParams<double, JitWords> p;
    rc = fill_view_params(p, words, nwords, out, n, exclusive, init_host, carry_host, carry_dev, seg_total_dev,
                          carry_out_dev, scratch, scratch_bytes, need, what);
    if (!rc) rc = launch_view_scan(k, p, vec_ok, device, (cudaStream_t)stream);
  } else if (acc_bytes == 4) {
    ScanParams<float, JitWords> p;
    rc = fill_view_params(p, words, nwords, out, n, exclusive, init_host, carry_host, carry_dev, seg_total_dev,
                          carry_out_dev, scratch, scratch_bytes, need, what);
    if (!rc) rc = launch_view_scan(k, p, vec_ok, device, (cudaStream_t)stream);
  } else {
    rc = set_error(DRK_E_ARG, "drk_jit_scan_view: acc_bytes must be 4 or 8");
  }
  g_chain_launch = 0;
  if (rc) return rc;
  return epilogue(what);
}

