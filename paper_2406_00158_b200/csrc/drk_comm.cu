// drk_comm.cu — the cross-GPU combine of a reduce in one process (reference
// algorithms.py:146-149, the driver's ascending fold of per-segment partials), on the
// device: a fold kernel over per-segment partials that live in device memory (the GPU's
// own slots, peer memory over NVLink, or an all-gathered buffer), and a single-process
// NCCL communicator (ncclCommInitAll over the runtime's GPUs) whose all-gather gives every
// GPU every partial, so each GPU folds the same value in the same order (an all-reduce
// whose result does not depend on NCCL's reduction order).
//
// NCCL is resolved at run time (dlopen of libnccl.so.2 — in a torch process that is the
// library torch already loaded), so libdrk.so has no link-time NCCL dependency and the
// rest of the library works where NCCL is absent (drk_comm_available() == 0).
#include <dlfcn.h>

#include "drk_host.h"

using namespace drk;
using namespace drk_host;

namespace {

// ---- NCCL, resolved at run time ------------------------------------------------------
typedef struct ncclComm* ncclComm_t;
typedef int ncclResult_t;
enum { NCCL_UINT64 = 5 };  // ncclUint64 (nccl.h)
struct Nccl {
  bool tried = false;
  void* so = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
  std::string why;
};
Nccl g_nccl;
std::mutex g_nccl_mu;

bool nccl_load() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.tried) return g_nccl.so != nullptr;
  g_nccl.tried = true;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* nm : names) {
    g_nccl.so = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (g_nccl.so) break;
  }
  if (!g_nccl.so) {
    const char* e = dlerror();
    g_nccl.why = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
    return false;
  }
  bool ok = true;
  auto sym = [&](const char* nm) {
    void* f = dlsym(g_nccl.so, nm);
    if (!f) ok = false;
    return f;
  };
  g_nccl.CommInitAll = (decltype(g_nccl.CommInitAll))sym("ncclCommInitAll");
  g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))sym("ncclCommDestroy");
  g_nccl.AllGather = (decltype(g_nccl.AllGather))sym("ncclAllGather");
  g_nccl.GroupStart = (decltype(g_nccl.GroupStart))sym("ncclGroupStart");
  g_nccl.GroupEnd = (decltype(g_nccl.GroupEnd))sym("ncclGroupEnd");
  g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))sym("ncclGetErrorString");
  g_nccl.GetVersion = (decltype(g_nccl.GetVersion))sym("ncclGetVersion");
  if (!ok) {
    g_nccl.why = "libnccl.so.2 lacks a required symbol";
    dlclose(g_nccl.so);
    g_nccl.so = nullptr;
    return false;
  }
  return true;
}

int nccl_status(ncclResult_t r, const char* what) {
  if (r == 0) return 0;
  const char* msg = g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?";
  return set_error(DRK_E_COMM, std::string(what) + ": NCCL error " + std::to_string(r) + " (" + msg + ")");
}

struct Comm {
  int ndev = 0;
  int devices[DRK_COMM_MAX_DEV];
  ncclComm_t comms[DRK_COMM_MAX_DEV];
};

// ---- the fold -------------------------------------------------------------------------
struct FoldArgs {
  const void* part[DRK_FOLD_MAX];
};

// acc = init; acc = acc ⊕ P(partial_k) for k = 0..count-1, in P (one thread: count <= 64)
template <class T, class Op>
__global__ void reduce_fold_kernel(const FoldArgs a, int count, typename PartialOf<T, Op>::type init,
                                   typename PartialOf<T, Op>::type* out_dev, typename PartialOf<T, Op>::type* out_host) {
  typedef typename WideAcc<T, Op>::type A;
  typedef typename PartialOf<T, Op>::type P;
  P acc = init;
  for (int k = 0; k < count; ++k) {
    const P v = (P) * (const A*)a.part[k];
    acc = Op::apply(acc, v);
  }
  if (out_dev) *out_dev = acc;
  if (out_host) *out_host = acc;
}

template <class T, class Op>
int reduce_fold_t(const FoldArgs& a, int count, const void* init, void* out_dev, void* out_host, cudaStream_t s) {
  typedef typename PartialOf<T, Op>::type P;
  P iv;
  memcpy(&iv, init, sizeof(P));
  reduce_fold_kernel<T, Op><<<1, 1, 0, s>>>(a, count, iv, (P*)out_dev, (P*)out_host);
  return 0;
}

template <class T>
int reduce_fold_op(int op, const FoldArgs& a, int count, const void* init, void* out_dev, void* out_host,
                   cudaStream_t s) {
  switch (op) {
    case DRK_ADD: return reduce_fold_t<T, OpAdd>(a, count, init, out_dev, out_host, s);
    case DRK_MUL: return reduce_fold_t<T, OpMul>(a, count, init, out_dev, out_host, s);
    case DRK_MIN: return reduce_fold_t<T, OpMin>(a, count, init, out_dev, out_host, s);
    case DRK_MAX: return reduce_fold_t<T, OpMax>(a, count, init, out_dev, out_host, s);
  }
  return set_error(DRK_E_ARG, "drk_reduce_fold: unknown op");
}

}  // namespace

extern "C" int drk_partial_dtype(int dtype, int op) {
  if (dtype == DRK_F32 || dtype == DRK_F64) return dtype;
  return drk_acc_dtype(dtype, op);
}

extern "C" int drk_reduce_fold(int dtype, int op, const void* const* partials, int count, const void* init,
                               void* result_dev, void* result_host_mapped, int device, void* stream) {
  const char* what = "drk_reduce_fold";
  if (count < 0 || count > DRK_FOLD_MAX) return set_error(DRK_E_ARG, "drk_reduce_fold: count out of range");
  if (count > 0 && !partials) return set_error(DRK_E_ARG, "drk_reduce_fold: null partials");
  if (!init) return set_error(DRK_E_ARG, "drk_reduce_fold: null init");
  if (!result_dev && !result_host_mapped) return set_error(DRK_E_ARG, "drk_reduce_fold: no result address");
  FoldArgs a;
  memset(&a, 0, sizeof(a));
  for (int k = 0; k < count; ++k) {
    if (!partials[k]) return set_error(DRK_E_ARG, "drk_reduce_fold: null partial");
    a.part[k] = partials[k];
  }
  if (int rc = prologue(device, what)) return rc;
  int rc = 0;
  switch (dtype) {
    case DRK_F32: rc = reduce_fold_op<float>(op, a, count, init, result_dev, result_host_mapped, (cudaStream_t)stream); break;
    case DRK_F64: rc = reduce_fold_op<double>(op, a, count, init, result_dev, result_host_mapped, (cudaStream_t)stream); break;
    case DRK_I32: rc = reduce_fold_op<int>(op, a, count, init, result_dev, result_host_mapped, (cudaStream_t)stream); break;
    case DRK_I64: rc = reduce_fold_op<long long>(op, a, count, init, result_dev, result_host_mapped, (cudaStream_t)stream); break;
    default: return set_error(DRK_E_DTYPE, "drk_reduce_fold: unknown dtype");
  }
  if (rc) return rc;
  drk_note_launch();
  return epilogue(what);
}

extern "C" int drk_comm_available(void) { return nccl_load() ? 1 : 0; }

extern "C" int drk_comm_version(void) {
  if (!nccl_load()) return 0;
  int v = 0;
  g_nccl.GetVersion(&v);
  return v;
}

extern "C" int drk_comm_create(int ndev, const int* devices, void** comm) {
  if (!comm) return set_error(DRK_E_ARG, "drk_comm_create: null comm");
  *comm = nullptr;
  if (ndev < 1 || ndev > DRK_COMM_MAX_DEV || !devices)
    return set_error(DRK_E_ARG, "drk_comm_create: ndev out of range");
  for (int i = 0; i < ndev; ++i)
    for (int j = 0; j < i; ++j)
      if (devices[i] == devices[j]) return set_error(DRK_E_ARG, "drk_comm_create: duplicate device");
  if (!nccl_load()) return set_error(DRK_E_COMM, "drk_comm_create: " + g_nccl.why);
  int cur = 0;
  cudaGetDevice(&cur);
  Comm* c = new Comm();
  c->ndev = ndev;
  for (int i = 0; i < ndev; ++i) c->devices[i] = devices[i];
  const ncclResult_t r = g_nccl.CommInitAll(c->comms, ndev, devices);
  cudaSetDevice(cur);
  if (r != 0) {
    delete c;
    return nccl_status(r, "drk_comm_create: ncclCommInitAll");
  }
  *comm = c;
  return 0;
}

extern "C" int drk_comm_destroy(void* comm) {
  if (!comm) return 0;
  Comm* c = (Comm*)comm;
  int rc = 0;
  for (int i = 0; i < c->ndev; ++i) {
    const ncclResult_t r = g_nccl.CommDestroy(c->comms[i]);
    if (r != 0 && rc == 0) rc = nccl_status(r, "drk_comm_destroy");
  }
  delete c;
  return rc;
}

extern "C" int drk_comm_allgather(void* comm, const void* const* send, void* const* recv, size_t words,
                                  void* const* streams) {
  if (!comm || !send || !recv || !streams) return set_error(DRK_E_ARG, "drk_comm_allgather: null argument");
  Comm* c = (Comm*)comm;
  if (words == 0) return 0;
  int cur = 0;
  cudaGetDevice(&cur);
  int rc = nccl_status(g_nccl.GroupStart(), "drk_comm_allgather: ncclGroupStart");
  if (rc) return rc;
  for (int i = 0; i < c->ndev && rc == 0; ++i) {
    cudaSetDevice(c->devices[i]);
    rc = nccl_status(g_nccl.AllGather(send[i], recv[i], words, NCCL_UINT64, c->comms[i], (cudaStream_t)streams[i]),
                     "drk_comm_allgather: ncclAllGather");
  }
  const int rc_end = nccl_status(g_nccl.GroupEnd(), "drk_comm_allgather: ncclGroupEnd");
  cudaSetDevice(cur);
  return rc ? rc : rc_end;
}

// The whole cross-GPU combine of one reduce: an all-gather of every GPU's `words` 8-byte
// partial slots (slots[i] on GPU i, padded to the same count), then on every GPU the fold of
// the gathered partials in segment order (order[k] = gathered slot of segment k) from init.
// Every GPU ends with the result in result_dev[i] (nullable array); GPU 0 also stores it into
// result_host_mapped.  One call, no host round trip.
extern "C" int drk_comm_reduce(void* comm, int dtype, int op, const void* const* slots, void* const* gather,
                               size_t words, const int* order, int count, const void* init, void* const* result_dev,
                               void* result_host_mapped, void* const* streams) {
  if (!comm || !slots || !gather || !streams || !init || (count > 0 && !order))
    return set_error(DRK_E_ARG, "drk_comm_reduce: null argument");
  Comm* c = (Comm*)comm;
  if (count < 0 || count > DRK_FOLD_MAX) return set_error(DRK_E_ARG, "drk_comm_reduce: count out of range");
  for (int k = 0; k < count; ++k)
    if (order[k] < 0 || (size_t)order[k] >= words * (size_t)c->ndev)
      return set_error(DRK_E_ARG, "drk_comm_reduce: order out of range");
  if (int rc = drk_comm_allgather(comm, slots, gather, words, streams)) return rc;
  for (int i = 0; i < c->ndev; ++i) {
    const void* parts[DRK_FOLD_MAX];
    for (int k = 0; k < count; ++k) parts[k] = (const char*)gather[i] + 8 * (size_t)order[k];
    void* rd = result_dev ? result_dev[i] : nullptr;
    void* rh = i == 0 ? result_host_mapped : nullptr;
    if (!rd && !rh) continue;
    if (int rc = drk_reduce_fold(dtype, op, parts, count, init, rd, rh, c->devices[i], streams[i])) return rc;
  }
  return 0;
}

// ---- one process per GPU: an all-gather of (has, value) pairs over peer memory ------------
// Each rank owns a mailbox (2 banks x world slots of 32 bytes: has, value, epoch, pad) in its GPU's
// memory, allocated here and exported with a CUDA IPC handle; every rank maps every other
// rank's mailbox (NVLink peer memory; cudaIpcMemLazyEnablePeerAccess).  One exchange is one
// kernel per rank: it stores the rank's pair into slot `rank` of every mailbox (peer stores,
// then a system-scope fence, then the slot's epoch word), waits until every slot of its own
// mailbox carries this epoch, and copies the pairs into `gathered` (16 bytes per rank, the
// layout an NCCL all-gather of the pairs produces).  The reduce's and the scan's cross-rank
// combine then need no NCCL call and no host.  A rank that never arrives does not hang the
// GPU: the wait gives up after timeout_ns and writes 1 into *status (0 on success).

extern "C" int drk_ipc_alloc(size_t bytes, int device, void** dev_ptr) {
  if (!dev_ptr || !bytes) return set_error(DRK_E_ARG, "drk_ipc_alloc: bad argument");
  *dev_ptr = nullptr;
  if (int rc = prologue(device, "drk_ipc_alloc")) return rc;
  DRK_CHECK(cudaMalloc(dev_ptr, bytes));  // a whole allocation: its IPC handle maps its base
  DRK_CHECK(cudaMemset(*dev_ptr, 0, bytes));
  return 0;
}

extern "C" int drk_ipc_free(void* dev_ptr) {
  if (dev_ptr) DRK_CHECK(cudaFree(dev_ptr));
  return 0;
}

extern "C" int drk_ipc_handle(void* dev_ptr, void* handle_out) {
  if (!dev_ptr || !handle_out) return set_error(DRK_E_ARG, "drk_ipc_handle: null argument");
  cudaIpcMemHandle_t h;
  DRK_CHECK(cudaIpcGetMemHandle(&h, dev_ptr));
  memcpy(handle_out, &h, sizeof(h));
  return 0;
}

extern "C" int drk_ipc_open(const void* handle, int device, void** dev_ptr) {
  if (!handle || !dev_ptr) return set_error(DRK_E_ARG, "drk_ipc_open: null argument");
  *dev_ptr = nullptr;
  if (int rc = prologue(device, "drk_ipc_open")) return rc;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  DRK_CHECK(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return 0;
}

extern "C" int drk_ipc_close(void* dev_ptr) {
  if (dev_ptr) DRK_CHECK(cudaIpcCloseMemHandle(dev_ptr));
  return 0;
}

namespace {
struct Mailboxes {
  unsigned long long* box[DRK_COMM_MAX_RANKS];
};

__global__ void mailbox_allgather_kernel(const unsigned long long* __restrict__ pair, const Mailboxes mb, int world,
                                         int rank, const volatile unsigned long long* own, unsigned long long epoch,
                                         unsigned long long timeout_ns, unsigned long long* gathered, int* status) {
  // two banks alternate by epoch: a rank that finished exchange e may already publish e + 1
  // before a slower rank has read exchange e, but not e + 2 (that needs the slower rank's e + 1)
  const int bank = (int)(epoch & 1ull) * world;
  const int j = threadIdx.x;
  if (j < world) {  // publish: the pair, then (after a system fence) this exchange's epoch
    unsigned long long* slot = mb.box[j] + 4 * (bank + rank);
    slot[0] = pair[0];
    slot[1] = pair[1];
    __threadfence_system();
    *(volatile unsigned long long*)(slot + 2) = epoch;
  }
  __syncwarp();
  int ok = 1;
  if (j < world) {
    unsigned long long t0, now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    const volatile unsigned long long* mine = own + 4 * (bank + j);
    while (mine[2] != epoch) {
      __nanosleep(128);
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (now - t0 > timeout_ns) {
        ok = 0;
        break;
      }
    }
    __threadfence_system();
    gathered[2 * j] = ok ? mine[0] : 0ull;
    gathered[2 * j + 1] = ok ? mine[1] : 0ull;
  }
  const int all = __all_sync(0xffffffffu, ok);
  if (j == 0) *status = all ? 0 : 1;
}
}  // namespace

extern "C" int drk_mailbox_allgather(const void* pair, void* const* peer_boxes, int world, int rank, const void* own_box,
                                     uint64_t epoch, uint64_t timeout_ns, void* gathered, void* status, int device,
                                     void* stream) {
  if (!pair || !peer_boxes || !own_box || !gathered || !status)
    return set_error(DRK_E_ARG, "drk_mailbox_allgather: null argument");
  if (world < 1 || world > DRK_COMM_MAX_RANKS || rank < 0 || rank >= world)
    return set_error(DRK_E_ARG, "drk_mailbox_allgather: rank / world out of range");
  Mailboxes mb;
  memset(&mb, 0, sizeof(mb));
  for (int j = 0; j < world; ++j) {
    if (!peer_boxes[j]) return set_error(DRK_E_ARG, "drk_mailbox_allgather: null mailbox");
    mb.box[j] = (unsigned long long*)peer_boxes[j];
  }
  if (int rc = prologue(device, "drk_mailbox_allgather")) return rc;
  mailbox_allgather_kernel<<<1, 32, 0, (cudaStream_t)stream>>>((const unsigned long long*)pair, mb, world, rank,
                                                               (const volatile unsigned long long*)own_box, epoch,
                                                               timeout_ns, (unsigned long long*)gathered, (int*)status);
  drk_note_launch();
  return epilogue("drk_mailbox_allgather");
}
