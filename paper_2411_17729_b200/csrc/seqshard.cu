// Sequence-sharded cascade (BASELINE configs[3] "per-stage NCCL halo
// exchange"), owned by the library: communicators, the halo exchange and its overlap with the
// stage GEMMs.
//
// Rank r of R owns time rows [r L_loc, (r+1) L_loc) of every sequence of ONE system. The cascade's
// stage k adds P_k v_{l-2^k}, so before stage k a rank needs the last 2^k time
// rows of v^(k) held by rank r-1 (zeros on rank 0: x_{-1} = 0). The fused first step
// v^(1) = Bbar u_l + Abar Bbar u_{l-1} needs one row of u, the fused last step
// y = C v + (C P_Ne) v_{l-2^Ne} + D u needs 2^Ne rows of v^(Ne) (R21).
//
// Layout: time-major. u_loc [L_loc][batch][p], y_loc [L_loc][batch][q], and the two state buffers
// [H + L_loc][batch][m] with H = 2^Ne halo rows in front: seen as one matrix of rows
// (l, b) -> l * batch + b, a time shift by s is a row shift by s * batch, and a halo of d time rows
// is ONE contiguous block of d * batch * m elements -- sent straight from the sender's state buffer
// and received straight into the receiver's halo rows (no packing, no copies).
//
// Per step, the GEMM (mimo_tc*.cu) runs in two launches: interior rows (l_loc >= s: every operand
// is local) first, then -- after the halo has landed -- the boundary rows [0, s). The exchange of
// step k's halo runs on the comm stream while step k-1's boundary launch and step k's interior
// launch run on the compute stream; it starts as soon as the rows it sends are written.
//
// Transports behind the same schedule:
//   NCCL   one rank per process and GPU: grouped ncclSend(r -> r+1) / ncclRecv(r-1 -> r) on the
//          comm stream (NVLink / NVSwitch on a B200 box). libnccl is resolved at run time (the copy
//          torch already loaded, else the system one); casc_comm_init fails with CASC_ERR_NCCL
//          when it is missing.
//   local  R emulated ranks in one process on one device (tests): each rank's apply runs on its own
//          host thread and streams; a halo is a device copy ordered by CUDA events, with a host
//          rendezvous per exchange. Ranks never spin on each other inside a kernel.
//
// CASC_HALO_PEER (apply_peer below): no halo copies at all -- the GEMM producing v^(k) stores its
// last 2^k rows ALSO into rank r+1's halo rows (epilogue of the CTA-pair kernels, over a peer
// mapping of rank r+1's workspace: CUDA IPC between NCCL ranks, the plain pointer between emulated
// ranks), and the transport carries only 1-byte ordering tokens.
#include <cuda.h>
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "engine.cuh"
#include "kernels.cuh"
#include "mimo_tc.cuh"
#include "profile.cuh"

namespace casc {

// ------------------------------------------------------------------------------ NCCL (run time)
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    // the copy already in the process (torch's), else whatever the loader finds
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))dlsym(h, "ncclCommInitRank");
    a.CommDestroy = (decltype(a.CommDestroy))dlsym(h, "ncclCommDestroy");
    a.Send = (decltype(a.Send))dlsym(h, "ncclSend");
    a.Recv = (decltype(a.Recv))dlsym(h, "ncclRecv");
    a.GroupStart = (decltype(a.GroupStart))dlsym(h, "ncclGroupStart");
    a.GroupEnd = (decltype(a.GroupEnd))dlsym(h, "ncclGroupEnd");
    a.GetErrorString = (decltype(a.GetErrorString))dlsym(h, "ncclGetErrorString");
    a.AllReduce = (decltype(a.AllReduce))dlsym(h, "ncclAllReduce");
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.Send && a.Recv && a.GroupStart && a.GroupEnd;
    return a;
  }();
  return api;
}

#define CASC_NCCL(x)                                                                          \
  do {                                                                                        \
    ncclResult_t r_ = (x);                                                                    \
    if (r_ != ncclSuccess) {                                                                  \
      if (getenv("CASC_DEBUG"))                                                               \
        fprintf(stderr, "casc: %s failed: %s\n", #x,                                          \
                nccl().GetErrorString ? nccl().GetErrorString(r_) : "?");                     \
      return CASC_ERR_NCCL;                                                                   \
    }                                                                                         \
  } while (0)

// ------------------------------------------------------------------------------ local transport
// Mailboxes of one emulated group: post(from, to, tag) -> (pointer, event) and a completion event
// back. Keys are (receiver or sender rank, exchange tag); entries live until the group is freed.
struct LocalGroup {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  struct Post { const void* src = nullptr; size_t bytes = 0; cudaEvent_t ready = nullptr; };
  std::map<std::pair<int, long>, Post> sends;          // keyed by receiving rank
  std::map<std::pair<int, long>, cudaEvent_t> copied;  // keyed by sending rank
  std::map<std::pair<int, long>, void*> ws_posts;      // CASC_HALO_PEER: each rank's workspace
  std::vector<cudaEvent_t> owned;
  ~LocalGroup() {
    for (auto e : owned) cudaEventDestroy(e);
  }
};

// how long an emulated rank waits for its neighbour to enqueue an exchange before reporting the
// group broken (CASC_ERR_NCCL): only host enqueue progress is awaited, never device work
static constexpr std::chrono::seconds kRendezvous{300};

struct Comm {
  int kind = 0;                 // 0 NCCL, 1 local
  int rank = 0, world = 1;
  ncclComm_t nc = nullptr;
  std::shared_ptr<LocalGroup> grp;
  long tag = 0;                 // exchanges issued by this rank (same sequence on every rank)
  // CASC_HALO_PEER between NCCL ranks: IPC mappings of the successor's workspaces (opened once per
  // allocation, closed by casc_comm_destroy) and a small device scratch for the handle exchange
  std::vector<std::pair<cudaIpcMemHandle_t, void*>> ipc;
  void* scratch = nullptr;
};

// One halo exchange on the comm stream `cs`: send `sbytes` from `sbuf` to rank+dir (if any),
// receive `rbytes` into `rbuf` from rank-dir (if any); dir = +1 (the halo direction) or -1.
// `after` (may be null) orders the send after the producing work; returns with an event on `cs`
// recorded in `done` (the exchange finished).
static int exchange(Comm* c, const void* sbuf, size_t sbytes, void* rbuf, size_t rbytes, cudaEvent_t after,
                    cudaStream_t cs, cudaEvent_t done, int dir = 1) {
  if (after) CASC_TRY(cudaStreamWaitEvent(cs, after, 0));
  const int to = c->rank + dir, from = c->rank - dir;
  const bool send = to >= 0 && to < c->world, recv = from >= 0 && from < c->world;
  const long tag = c->tag++;
  if (c->kind == 0) {
    if (send || recv) {
      const NcclApi& n = nccl();
      CASC_NCCL(n.GroupStart());
      if (send) CASC_NCCL(n.Send(sbuf, sbytes, ncclUint8, to, c->nc, cs));
      if (recv) CASC_NCCL(n.Recv(rbuf, rbytes, ncclUint8, from, c->nc, cs));
      CASC_NCCL(n.GroupEnd());
    }
  } else {
    LocalGroup& g = *c->grp;
    if (send) {                                          // publish: where the rows are, and when
      cudaEvent_t ready;
      CASC_TRY(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
      CASC_TRY(cudaEventRecord(ready, cs));
      std::lock_guard<std::mutex> lk(g.mu);
      g.owned.push_back(ready);
      g.sends[{to, tag}] = LocalGroup::Post{sbuf, sbytes, ready};
      g.cv.notify_all();
    }
    if (recv) {                                          // wait for rank-dir's post, copy, report back
      LocalGroup::Post p;
      {
        std::unique_lock<std::mutex> lk(g.mu);
        // a neighbour that failed before posting would leave this rank waiting: bounded wait
        if (!g.cv.wait_for(lk, kRendezvous, [&] { return g.sends.count({c->rank, tag}) > 0; })) return CASC_ERR_NCCL;
        p = g.sends[{c->rank, tag}];
      }
      if (p.bytes != rbytes) return CASC_ERR_DIM;
      CASC_TRY(cudaStreamWaitEvent(cs, p.ready, 0));
      CASC_TRY(cudaMemcpyAsync(rbuf, p.src, rbytes, cudaMemcpyDeviceToDevice, cs));
      cudaEvent_t cp;
      CASC_TRY(cudaEventCreateWithFlags(&cp, cudaEventDisableTiming));
      CASC_TRY(cudaEventRecord(cp, cs));
      std::lock_guard<std::mutex> lk(g.mu);
      g.owned.push_back(cp);
      g.copied[{from, tag}] = cp;
      g.cv.notify_all();
    }
    if (send) {                                          // the send completes when rank+dir has copied
      cudaEvent_t cp;
      {
        std::unique_lock<std::mutex> lk(g.mu);
        if (!g.cv.wait_for(lk, kRendezvous, [&] { return g.copied.count({c->rank, tag}) > 0; })) return CASC_ERR_NCCL;
        cp = g.copied[{c->rank, tag}];
      }
      CASC_TRY(cudaStreamWaitEvent(cs, cp, 0));
    }
  }
  CASC_TRY(cudaEventRecord(done, cs));
  return CASC_OK;
}

// ------------------------------------------------------------------------------ workspace
struct SeqWs {
  MimoWs mw;           // derived weights (no state buffers: L = 0)
  void* u_edge;        // [(uh + Bu) batch][p]: the u halo (uh time rows) + the first Bu local rows of u
  void *Va, *Vb;       // [(H + L_loc) * batch][m]
  char* tok;           // CASC_HALO_PEER ordering tokens: [0] sent, [128] received
  size_t bytes;
};
static constexpr int64_t kRowBlock = 256;            // boundary granularity: one CTA-pair tile

// boundary rows of a step with time shift s: the row blocks that read rows l - s < 0
static int64_t boundary_rows(int64_t s, int batch, int64_t rows) {
  return std::min(rows, ceil_div(s * batch, kRowBlock) * kRowBlock);
}

// time rows of u the first step reads before l: 3 for the Krylov head (Ne >= 2, lags 0..3, R28),
// else 1 (the fused first step, or y directly when Ne = 0)
static int u_halo_rows(int Ne) { return Ne >= 2 ? 3 : 1; }

static SeqWs carve_seq(void* ws, int m, int p, int q, int64_t L_loc, int batch, int Ne, int mode) {
  SeqWs w{};
  w.mw = carve_mimo(ws, m, p, q, 0, 0, mode);
  Carver c(ws);
  c.off = w.mw.bytes;
  const size_t es = mode == CASC_FP32 ? 4 : 2;
  const int64_t rows = L_loc * batch, H = mimo_out_halo(Ne);
  const int uh = u_halo_rows(Ne);
  const int64_t Bu = boundary_rows(uh, batch, rows);
  w.u_edge = c.take<char>((size_t)(uh * batch + Bu) * p * es);
  w.Va = c.take<char>((size_t)(H * batch + rows) * m * es);
  w.Vb = c.take<char>((size_t)(H * batch + rows) * m * es);
  w.tok = c.take<char>(256);
  w.bytes = c.bytes();
  return w;
}

// A row range [0, rows) of one step as a MIMO GEMM over the time-major matrix (batch folded into
// the rows): sources get row shifts s * batch; t_first skips the boundary tiles.
static int step_gemm(MimoGemm g, int64_t rows, int t_first, bool tf32, cudaStream_t st) {
  g.L = rows;
  g.batch = 1;
  g.t_first = t_first;
  return launch_mimo_gemm(g, tf32, st);
}

// NEXT-2, one-shot u halo: the cascade is a polynomial of degree 2^(Ne+1) - 1 in the shift
// (PAPER.md:137-141), so the local outputs need exactly Hu = 2^(Ne+1) - 1 time rows of u before the
// shard (pin T14: the windowed cascade equals the global one). One exchange of those rows, then
// the whole cascade runs on the extended window [l0 - Hu, l0 + L_loc) with no further
// communication; y is formed on the local rows only.
struct OneShotWs {
  MimoWs mw;
  void* u_ext;         // [(Hu + L_loc) batch][p]
  void *Va, *Vb;       // [(Hu + L_loc) batch][m]
  size_t bytes;
};
static int64_t oneshot_halo_rows(int Ne) { return Ne > 0 ? ((int64_t)2 << Ne) - 1 : 1; }
static OneShotWs carve_oneshot(void* ws, int m, int p, int q, int64_t L_loc, int batch, int Ne, int mode) {
  OneShotWs w{};
  w.mw = carve_mimo(ws, m, p, q, 0, 0, mode);
  Carver c(ws);
  c.off = w.mw.bytes;
  const size_t es = mode == CASC_FP32 ? 4 : 2;
  const int64_t ext = (oneshot_halo_rows(Ne) + L_loc) * batch;
  w.u_ext = c.take<char>((size_t)ext * p * es);
  w.Va = c.take<char>((size_t)ext * m * es);
  w.Vb = c.take<char>((size_t)ext * m * es);
  w.bytes = c.bytes();
  return w;
}

static int apply_oneshot(Comm* c, int m, int p, int q, int64_t L_loc, int batch, int Ne, int N_max, int mode,
                         const PackLayout& P, const double* Bbar, const double* C, const double* D, const void* u_loc,
                         void* y_loc, void* ws, size_t ws_bytes, cudaStream_t st, cudaStream_t cs) {
  OneShotWs w = carve_oneshot(ws, m, p, q, L_loc, batch, Ne, mode);
  if (ws_bytes < w.bytes) return CASC_ERR_WORKSPACE;
  const bool tf32 = mode == CASC_FP32;
  const size_t es = tf32 ? 4 : 2;
  const int64_t Hu = oneshot_halo_rows(Ne), rows = L_loc * batch, hr = Hu * batch, ext = hr + rows;
  const int64_t mm = (int64_t)m * m;
  int rc;
  if ((rc = mimo_derive(m, p, q, Ne, P, Bbar, C, D, w.mw, tf32, st))) return rc;
  cudaEvent_t ev_in = nullptr, ev_halo = nullptr;
  struct EvFree {
    cudaEvent_t* a; cudaEvent_t* b;
    ~EvFree() { if (*a) cudaEventDestroy(*a); if (*b) cudaEventDestroy(*b); }
  } ev_free{&ev_in, &ev_halo};
  CASC_TRY(cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming));
  CASC_TRY(cudaEventCreateWithFlags(&ev_halo, cudaEventDisableTiming));
  // the window: Hu rows of rank r-1's u (zeros on rank 0), then the local rows
  CASC_TRY(cudaMemsetAsync(w.u_ext, 0, (size_t)hr * p * es, st));
  CASC_TRY(cudaMemcpyAsync((char*)w.u_ext + (size_t)hr * p * es, u_loc, (size_t)rows * p * es,
                           cudaMemcpyDeviceToDevice, st));
  CASC_TRY(cudaEventRecord(ev_in, st));
  {
    CASC_TRY(cudaStreamWaitEvent(cs, ev_in, 0));
    ProfScope ps(cs, K_SEQ_HALO, 2.0 * hr * p * es, 0.0);
    if ((rc = exchange(c, (const char*)u_loc + (size_t)(rows - hr) * p * es, (size_t)hr * p * es, w.u_ext,
                       (size_t)hr * p * es, nullptr, cs, ev_halo)))
      return rc;
  }
  CASC_TRY(cudaStreamWaitEvent(st, ev_halo, 0));
  const double dr = (double)ext;
  const int pipe = tf32 ? PIPE_TF32 : PIPE_BF16;
  const double xf = tf32 ? 3.0 : 1.0;
  auto run = [&](MimoGemm g, int64_t n_rows, int cls, double bytes, double flops) -> int {
    ProfScope ps(st, cls, bytes, flops);
    ps.exec(bytes, xf * flops, pipe);
    return step_gemm(g, n_rows, 0, tf32, st);
  };
  if (Ne == 0) {                       // y = (C Bbar + D) u_l + (C Abar Bbar) u_{l-1}, local rows
    MimoGemm g{};
    g.src[0] = {w.u_ext, w.mw.CBD, p, 0};
    g.src[1] = {w.u_ext, w.mw.CAB, p, batch};
    g.src[0].row0 = g.src[1].row0 = hr;
    g.n_src = 2; g.out = y_loc; g.n_out = q;
    return run(g, rows, K_MIMO_LAST, (double)rows * (p + q) * es, (double)rows * 4.0 * q * p);
  }
  const int k0 = Ne >= 2 ? 2 : 1;
  {                                    // head (Ne >= 2, R28) or fused first step over the window
    const void* Wj[4] = {w.mw.Bb, w.mw.AB, w.mw.A2B, w.mw.A3B};
    MimoGemm g{};
    g.n_src = Ne >= 2 ? 4 : 2;
    for (int j = 0; j < g.n_src; ++j) g.src[j] = {w.u_ext, Wj[j], p, (int64_t)j * batch};
    g.out = k0 == 2 ? w.Vb : w.Va; g.n_out = m;
    if ((rc = run(g, ext, K_MIMO_FIRST, dr * (p + m) * es, dr * 2.0 * g.n_src * m * p))) return rc;
  }
  const int kl = mimo_fold(Ne) ? Ne - 1 : Ne;   // the level the output step reads (R31)
  for (int k = k0; k <= kl - 1; ++k) {  // stages over the window (rows before it read zeros)
    void* Vs = (k - 1) % 2 == 0 ? w.Va : w.Vb;
    void* Vd = (k % 2 == 0) ? w.Va : w.Vb;
    const void* Wk = tf32 ? static_cast<const void*>(P.f32 + k * 2 * mm) : static_cast<const void*>(P.b16 + k * mm);
    MimoGemm g{};
    g.src[0] = {Vs, Wk, m, ((int64_t)1 << k) * batch};
    g.n_src = 1; g.R = Vs; g.out = Vd; g.n_out = m;
    if ((rc = run(g, ext, K_MIMO_STAGE, dr * m * es * 2.0, dr * 2.0 * (double)mm))) return rc;
  }
  void* V = (kl - 1) % 2 == 0 ? w.Va : w.Vb;   // y on the local rows from v^(kl) (R21 / R31) + D u
  MimoGemm g{};
  mimo_output_gemm(g, w.mw, Ne, m, p, q, V, hr, u_loc, 0, D != nullptr, batch);
  g.out = y_loc; g.n_out = q;
  const double k_in = (double)(g.n_src - (D ? 1 : 0)) * m + (D ? p : 0);
  return run(g, rows, K_MIMO_LAST, (double)rows * (m + p + q) * es, (double)rows * 2.0 * q * k_in);
}


// ------------------------------------------------------------------------------ CASC_HALO_PEER
// The successor's (rank + 1) workspace as a pointer this device can store into; null on the last
// rank. Emulated ranks post their ws pointers through the group. NCCL ranks send a CUDA IPC handle
// of their ws allocation (+ the offset of ws in it) to rank - 1 and map the one they receive (once
// per allocation, cached in the comm); an allreduce makes every rank agree that the mapping worked.
static int peer_ws(Comm* c, void* ws, cudaStream_t cs, void** succ) {
  *succ = nullptr;
  const long tag = c->tag++;
  if (c->kind == 1) {
    LocalGroup& g = *c->grp;
    std::unique_lock<std::mutex> lk(g.mu);
    g.ws_posts[{c->rank, tag}] = ws;
    g.cv.notify_all();
    if (c->rank + 1 < c->world) {
      if (!g.cv.wait_for(lk, kRendezvous, [&] { return g.ws_posts.count({c->rank + 1, tag}) > 0; })) return CASC_ERR_NCCL;
      *succ = g.ws_posts[{c->rank + 1, tag}];
    }
    return CASC_OK;
  }
  if (c->world == 1) return CASC_OK;
  const NcclApi& n = nccl();
  if (!n.AllReduce) return CASC_ERR_UNSUPPORTED;
  struct Msg { cudaIpcMemHandle_t h; uint64_t off; int32_t ok; int32_t pad; };
  static_assert(sizeof(Msg) <= 128, "scratch layout");
  if (!c->scratch) CASC_TRY(cudaMalloc(&c->scratch, 512));
  char* sc = static_cast<char*>(c->scratch);                 // [0] my msg, [128] successor's, [256] flag
  Msg mine{};
  {
    using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static GetRange get_range = [] {
      void* f = nullptr;
      cudaDriverEntryPointQueryResult q;
      return (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) == cudaSuccess &&
              q == cudaDriverEntryPointSuccess) ? reinterpret_cast<GetRange>(f) : nullptr;
    }();
    CUdeviceptr base = 0;
    size_t size = 0;
    if (get_range && get_range(&base, &size, (CUdeviceptr)ws) == CUDA_SUCCESS &&
        cudaIpcGetMemHandle(&mine.h, (void*)base) == cudaSuccess) {
      mine.off = (uint64_t)((CUdeviceptr)ws - base);
      mine.ok = 1;
    }
    cudaGetLastError();                                       // a VMM allocation has no IPC handle
  }
  CASC_TRY(cudaMemcpyAsync(sc, &mine, sizeof(mine), cudaMemcpyHostToDevice, cs));
  cudaEvent_t done;
  CASC_TRY(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
  int rc = exchange(c, sc, 128, sc + 128, 128, nullptr, cs, done, -1);   // to rank - 1, from rank + 1
  cudaEventDestroy(done);
  if (rc) return rc;
  Msg theirs{};
  if (c->rank + 1 < c->world) CASC_TRY(cudaMemcpyAsync(&theirs, sc + 128, sizeof(theirs), cudaMemcpyDeviceToHost, cs));
  CASC_TRY(cudaStreamSynchronize(cs));
  int ok = 1;
  if (c->rank + 1 < c->world) {
    ok = theirs.ok;
    if (ok) {
      void* mapped = nullptr;
      for (auto& e : c->ipc)
        if (!memcmp(&e.first, &theirs.h, sizeof(theirs.h))) mapped = e.second;
      if (!mapped) {
        if (cudaIpcOpenMemHandle(&mapped, theirs.h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess) {
          c->ipc.emplace_back(theirs.h, mapped);
        } else {
          cudaGetLastError();
          mapped = nullptr;
          ok = 0;
        }
      }
      if (mapped) *succ = static_cast<char*>(mapped) + theirs.off;
    }
  }
  // every rank must take the same path: agree on the minimum
  int* flag = reinterpret_cast<int*>(sc + 256);
  CASC_TRY(cudaMemcpyAsync(flag, &ok, sizeof(int), cudaMemcpyHostToDevice, cs));
  CASC_NCCL(n.AllReduce(flag, flag, 1, ncclInt32, ncclMin, c->nc, cs));
  CASC_TRY(cudaMemcpyAsync(&ok, flag, sizeof(int), cudaMemcpyDeviceToHost, cs));
  CASC_TRY(cudaStreamSynchronize(cs));
  if (!ok) {
    *succ = nullptr;
    return CASC_ERR_UNSUPPORTED;
  }
  return CASC_OK;
}

// The per-stage schedule of casc_apply_seqsharded with the halo rows delivered by the producing
// GEMM itself (see the file header). Per step k, on rank r (stream order on st / cs):
//   interior launch of step k-1 (its epilogue stores v^(k)'s last 2^k rows into rank r+1's halo
//   rows) -> token "ready" to r+1 ... boundary launch of step k after "ready" from r-1 -> token
//   "consumed" to r-1; the next interior launch (which overwrites rank r+1's halo rows of the other
//   buffer) waits for "consumed" from r+1. One token exchange at the start ("my buffers are free")
//   covers the previous call. Every rank issues the same sequence of exchanges.
static int apply_peer(Comm* c, int m, int p, int q, int64_t L_loc, int batch, int Ne, int N_max, int mode,
                      const PackLayout& P, const double* Bbar, const double* C, const double* D, const void* u_loc,
                      void* y_loc, void* ws, size_t ws_bytes, cudaStream_t st, cudaStream_t cs) {
  SeqWs w = carve_seq(ws, m, p, q, L_loc, batch, Ne, mode);
  if (ws_bytes < w.bytes) return CASC_ERR_WORKSPACE;
  const bool tf32 = mode == CASC_FP32;
  const size_t es = tf32 ? 4 : 2;
  const int64_t rows = L_loc * batch, Hr = mimo_out_halo(Ne) * batch, mm = (int64_t)m * m;
  const int uh = u_halo_rows(Ne);
  const int k0 = Ne >= 2 ? 2 : 1, kl = mimo_fold(Ne) ? Ne - 1 : Ne;
  auto halo_time = [&](int k) -> int64_t { return k < kl ? ((int64_t)1 << k) : mimo_out_halo(Ne); };
  // every pushed row must come from an interior launch
  for (int k = k0; k <= kl; ++k) {
    const int64_t s_prev = k == k0 ? uh : ((int64_t)1 << (k - 1));
    if (rows - halo_time(k) * batch < boundary_rows(s_prev, batch, rows)) return CASC_ERR_UNSUPPORTED;
  }
  {                                                  // the state-producing GEMMs must be CTA-pair
    MimoGemm head{}, stage{};                        // kernels (decided alike on every rank)
    head.n_src = Ne >= 2 ? 4 : 2;
    for (int j = 0; j < head.n_src; ++j) head.src[j].K = p;
    head.n_out = m;
    stage.n_src = 1; stage.src[0].K = m; stage.n_out = m;
    auto pair = [&](const MimoGemm& g) { return mimo_pair_ok(g, tf32) || (tf32 && mimo_pair_tf32_ok(g)); };
    if (!pair(head) || (k0 < kl && !pair(stage))) return CASC_ERR_UNSUPPORTED;
  }
  int rc;
  void* succ = nullptr;
  if ((rc = peer_ws(c, ws, cs, &succ))) return rc;
  auto peer_of = [&](void* local) -> void* { return succ ? static_cast<char*>(succ) + (static_cast<char*>(local) - static_cast<char*>(ws)) : nullptr; };
  if ((rc = mimo_derive(m, p, q, Ne, P, Bbar, C, D, w.mw, tf32, st))) return rc;

  std::vector<cudaEvent_t> evs;
  struct EvFree {
    std::vector<cudaEvent_t>& v;
    ~EvFree() { for (auto e : v) cudaEventDestroy(e); }
  } ev_free{evs};
  auto new_event = [&](cudaEvent_t* e) -> int {
    CASC_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    evs.push_back(*e);
    return CASC_OK;
  };
  cudaEvent_t ev_in, ev_uhalo, ev_ack;
  if ((rc = new_event(&ev_in)) || (rc = new_event(&ev_uhalo)) || (rc = new_event(&ev_ack))) return rc;
  // rank 0's halo rows stay zero; the others are overwritten by rank r-1's pushes
  CASC_TRY(cudaMemsetAsync(w.Va, 0, (size_t)Hr * m * es, st));
  CASC_TRY(cudaMemsetAsync(w.Vb, 0, (size_t)Hr * m * es, st));
  const size_t uhb = (size_t)uh * batch * p * es;
  CASC_TRY(cudaMemsetAsync(w.u_edge, 0, uhb, st));
  const int64_t Bu = boundary_rows(uh, batch, rows);
  CASC_TRY(cudaMemcpyAsync((char*)w.u_edge + uhb, u_loc, (size_t)Bu * p * es, cudaMemcpyDeviceToDevice, st));
  CASC_TRY(cudaEventRecord(ev_in, st));
  {                                                  // the u halo (an input: exchanged as it is)
    CASC_TRY(cudaStreamWaitEvent(cs, ev_in, 0));
    ProfScope ps(cs, K_SEQ_HALO, 2.0 * uhb, 0.0);
    if ((rc = exchange(c, (const char*)u_loc + (size_t)(rows - (int64_t)uh * batch) * p * es, uhb, w.u_edge, uhb,
                       nullptr, cs, ev_uhalo)))
      return rc;
  }
  // "my halo rows are free": after the memsets (and everything before this call on st)
  if ((rc = exchange(c, w.tok, 1, w.tok + 128, 1, ev_in, cs, ev_ack, -1))) return rc;

  const double dr = (double)rows;
  const int pipe = tf32 ? PIPE_TF32 : PIPE_BF16;
  const double xf = tf32 ? 3.0 : 1.0;
  // interior rows of a step; with `push`, its output rows l >= rows - d also land in rank r+1's halo
  auto interior = [&](MimoGemm g, int64_t s_time, void* out_local, int64_t d_push, int cls, double bytes,
                      double flops) -> int {
    const int64_t Bs = boundary_rows(s_time, batch, rows);
    if (d_push > 0 && succ) {
      g.peer_out = peer_of(out_local);
      g.peer_l_begin = rows - d_push;
      g.peer_shift = rows;
    }
    CASC_TRY(cudaStreamWaitEvent(st, ev_ack, 0));    // rank r+1 has read what we overwrite
    ProfScope ps(st, cls, bytes * (dr - Bs) / dr, flops * (dr - Bs) / dr);
    ps.exec(bytes * (dr - Bs) / dr, xf * flops * (dr - Bs) / dr, pipe);
    return Bs < rows ? step_gemm(g, rows, (int)(Bs / 128), tf32, st) : CASC_OK;
  };
  auto boundary = [&](MimoGemm g, int64_t s_time, cudaEvent_t ready, int cls, double bytes, double flops) -> int {
    const int64_t Bs = boundary_rows(s_time, batch, rows);
    CASC_TRY(cudaStreamWaitEvent(st, ready, 0));
    ProfScope ps(st, cls, bytes * Bs / dr, flops * Bs / dr);
    ps.exec(bytes * Bs / dr, xf * flops * Bs / dr, pipe);
    return step_gemm(g, Bs, 0, tf32, st);
  };
  auto ready_token = [&](cudaEvent_t* ready) -> int {        // after the interior launch just queued
    cudaEvent_t after;
    int r2;
    if ((r2 = new_event(&after)) || (r2 = new_event(ready))) return r2;
    CASC_TRY(cudaEventRecord(after, st));
    return exchange(c, w.tok, 1, w.tok + 128, 1, after, cs, *ready, 1);
  };
  auto consumed_token = [&]() -> int {                        // after the boundary launch just queued
    cudaEvent_t after;
    int r2;
    if ((r2 = new_event(&after)) || (r2 = new_event(&ev_ack))) return r2;
    CASC_TRY(cudaEventRecord(after, st));
    return exchange(c, w.tok, 1, w.tok + 128, 1, after, cs, ev_ack, -1);
  };

  // ---- first step (Krylov head or fused first step): v^(k0), its last rows pushed to rank r+1
  void* Vhead = k0 == 2 ? w.Vb : w.Va;
  cudaEvent_t ready;
  {
    const void* Wj[4] = {w.mw.Bb, w.mw.AB, w.mw.A2B, w.mw.A3B};
    MimoGemm g{};
    g.n_src = Ne >= 2 ? 4 : 2;
    for (int j = 0; j < g.n_src; ++j) g.src[j] = {u_loc, Wj[j], p, (int64_t)j * batch};
    g.out = Vhead; g.out_row0 = Hr; g.n_out = m;
    MimoGemm gb = g;
    for (int j = 0; j < g.n_src; ++j) {
      gb.src[j] = {w.u_edge, Wj[j], p, (int64_t)j * batch};
      gb.src[j].row0 = uh * batch;
    }
    const double by = dr * (p + m) * es, fl = dr * 2.0 * g.n_src * m * p;
    if ((rc = interior(g, uh, Vhead, halo_time(k0) * batch, K_MIMO_FIRST, by, fl))) return rc;
    if ((rc = ready_token(&ready))) return rc;
    if ((rc = boundary(gb, uh, ev_uhalo, K_MIMO_FIRST, by, fl))) return rc;
  }
  // ---- steps k = k0 .. kl (the last one is the output step)
  for (int k = k0; k <= kl; ++k) {
    void* Vs = (k - 1) % 2 == 0 ? w.Va : w.Vb;       // holds v^(k), halo rows pushed by rank r-1
    void* Vd = (k % 2 == 0) ? w.Va : w.Vb;
    const int64_t d = halo_time(k) * batch;
    MimoGemm g{};
    cudaEvent_t next_ready = nullptr;
    double by, fl;
    int cls;
    if (k < kl) {
      const void* Wk = tf32 ? static_cast<const void*>(P.f32 + k * 2 * mm) : static_cast<const void*>(P.b16 + k * mm);
      g.src[0] = {Vs, Wk, m, d};
      g.src[0].row0 = Hr;
      g.n_src = 1; g.R = Vs; g.R_row0 = Hr; g.out = Vd; g.out_row0 = Hr; g.n_out = m;
      by = dr * m * es * 2.0; fl = dr * 2.0 * (double)mm; cls = K_MIMO_STAGE;
      if ((rc = interior(g, (int64_t)1 << k, Vd, halo_time(k + 1) * batch, cls, by, fl))) return rc;
      if ((rc = ready_token(&next_ready))) return rc;
    } else {
      mimo_output_gemm(g, w.mw, Ne, m, p, q, Vs, Hr, u_loc, 0, D != nullptr, batch);
      g.out = y_loc; g.n_out = q;
      const double k_in = (double)(g.n_src - (D ? 1 : 0)) * m + (D ? p : 0);
      by = dr * (m + p + q) * es; fl = dr * 2.0 * q * k_in; cls = K_MIMO_LAST;
      if ((rc = interior(g, halo_time(k), nullptr, 0, cls, by, fl))) return rc;
    }
    if ((rc = boundary(g, k < kl ? ((int64_t)1 << k) : halo_time(k), ready, cls, by, fl))) return rc;
    if ((rc = consumed_token())) return rc;
    ready = next_ready;
  }
  return CASC_OK;
}

}  // namespace casc

using namespace casc;
extern "C" {

int casc_nccl_unique_id(void* id_out) {
  if (!id_out) return CASC_ERR_ARG;
  if (!nccl().ok) return CASC_ERR_NCCL;
  ncclUniqueId id;
  CASC_NCCL(nccl().GetUniqueId(&id));
  memcpy(id_out, &id, sizeof(id));
  return CASC_OK;
}

int casc_comm_init(void** comm, int rank, int world, const void* nccl_unique_id) {
  if (!comm || !nccl_unique_id || world < 1 || rank < 0 || rank >= world) return CASC_ERR_ARG;
  *comm = nullptr;
  if (!nccl().ok) return CASC_ERR_NCCL;
  ncclUniqueId id;
  memcpy(&id, nccl_unique_id, sizeof(id));
  auto* c = new Comm();
  c->kind = 0;
  c->rank = rank;
  c->world = world;
  const ncclResult_t r = nccl().CommInitRank(&c->nc, world, id, rank);
  if (r != ncclSuccess) {
    if (getenv("CASC_DEBUG"))
      fprintf(stderr, "casc: ncclCommInitRank: %s\n", nccl().GetErrorString ? nccl().GetErrorString(r) : "?");
    delete c;
    return CASC_ERR_NCCL;
  }
  *comm = c;
  return CASC_OK;
}

int casc_comm_init_local(void** comms, int world) {
  if (!comms || world < 1) return CASC_ERR_ARG;
  auto grp = std::make_shared<LocalGroup>();
  grp->world = world;
  for (int r = 0; r < world; ++r) {
    auto* c = new Comm();
    c->kind = 1;
    c->rank = r;
    c->world = world;
    c->grp = grp;
    comms[r] = c;
  }
  return CASC_OK;
}

int casc_comm_destroy(void* comm) {
  if (!comm) return CASC_ERR_ARG;
  auto* c = static_cast<Comm*>(comm);
  int rc = CASC_OK;
  for (auto& e : c->ipc) cudaIpcCloseMemHandle(e.second);
  if (c->scratch) cudaFree(c->scratch);
  if (c->kind == 0 && c->nc && nccl().CommDestroy(c->nc) != ncclSuccess) rc = CASC_ERR_NCCL;
  delete c;
  return rc;
}

int casc_comm_rank(const void* comm, int* rank, int* world) {
  if (!comm) return CASC_ERR_ARG;
  auto* c = static_cast<const Comm*>(comm);
  if (rank) *rank = c->rank;
  if (world) *world = c->world;
  return CASC_OK;
}

size_t casc_apply_seqsharded_workspace(int m, int p, int q, int64_t L_loc, int batch, int N, int world, int mode,
                                       int halo) {
  if (m < 1 || p < 1 || q < 1 || L_loc < 1 || batch < 1 || N < 0 || world < 1) return 0;
  const int Ne = eff_order(N, L_loc * world);
  if (halo == CASC_HALO_ONESHOT_U) return carve_oneshot(nullptr, m, p, q, L_loc, batch, Ne, mode).bytes;
  return carve_seq(nullptr, m, p, q, L_loc, batch, Ne, mode).bytes;
}

int casc_apply_seqsharded(void* comm, int m, int p, int q, int64_t L_loc, int batch, int N, int N_max, int mode,
                          int halo, const void* pack, const double* Bbar, const double* C, const double* D,
                          const void* u_loc, void* y_loc, void* ws, size_t ws_bytes, void* compute_stream,
                          void* comm_stream) {
  g_launches = 0;
  auto* c = static_cast<Comm*>(comm);
  if (!c || !pack || !Bbar || !C || !u_loc || !y_loc || !ws || !comm_stream) return CASC_ERR_ARG;
  int rc = validate_common(1, m, p, q, L_loc, batch, N_max, mode);
  if (rc == kEmptyCall) return CASC_ERR_ARG;        // every rank owns at least one row and sequence
  if (rc) return rc;
  if (N < 0 || N > N_max) return CASC_ERR_DIM;
  if (!mimo_tc_supported(m, p, q)) return CASC_ERR_UNSUPPORTED;
  if (halo != CASC_HALO_PER_STAGE && halo != CASC_HALO_ONESHOT_U && halo != CASC_HALO_PEER) return CASC_ERR_ARG;
  const int64_t L = L_loc * c->world;
  const int Ne = eff_order(N, L);
  if (halo == CASC_HALO_PEER && Ne > 0) {
    if (c->world > 1 && (mimo_out_halo(Ne) > L_loc || u_halo_rows(Ne) > L_loc)) return CASC_ERR_UNSUPPORTED;
    return apply_peer(c, m, p, q, L_loc, batch, Ne, N_max, mode, pack_layout(const_cast<void*>(pack), 1, m, N_max, mode),
                      Bbar, C, D, u_loc, y_loc, ws, ws_bytes, (cudaStream_t)compute_stream, (cudaStream_t)comm_stream);
  }
  if (halo == CASC_HALO_ONESHOT_U) {
    // the Hu-row window must come from the immediate predecessor
    if (c->world > 1 && oneshot_halo_rows(Ne) > L_loc) return CASC_ERR_UNSUPPORTED;
    return apply_oneshot(c, m, p, q, L_loc, batch, Ne, N_max, mode,
                         pack_layout(const_cast<void*>(pack), 1, m, N_max, mode), Bbar, C, D, u_loc, y_loc, ws,
                         ws_bytes, (cudaStream_t)compute_stream, (cudaStream_t)comm_stream);
  }
  // each halo must come from the immediate predecessor (holds for configs[3] up to 8 ranks)
  const int uh = u_halo_rows(Ne);
  if (c->world > 1 && (mimo_out_halo(Ne) > L_loc || uh > L_loc)) return CASC_ERR_UNSUPPORTED;
  SeqWs w = carve_seq(ws, m, p, q, L_loc, batch, Ne, mode);
  if (ws_bytes < w.bytes) return CASC_ERR_WORKSPACE;
  cudaStream_t st = (cudaStream_t)compute_stream, cs = (cudaStream_t)comm_stream;
  const bool tf32 = mode == CASC_FP32;
  const size_t es = tf32 ? 4 : 2;
  const int64_t rows = L_loc * batch, H = mimo_out_halo(Ne), Hr = H * batch;
  PackLayout P = pack_layout(const_cast<void*>(pack), 1, m, N_max, mode);
  const int64_t mm = (int64_t)m * m;
  if ((rc = mimo_derive(m, p, q, Ne, P, Bbar, C, D, w.mw, tf32, st))) return rc;

  std::vector<cudaEvent_t> evs;
  struct EvFree {
    std::vector<cudaEvent_t>& v;
    ~EvFree() { for (auto e : v) cudaEventDestroy(e); }   // released once the device is done
  } ev_free{evs};
  auto new_event = [&](cudaEvent_t* e) -> int {
    CASC_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    evs.push_back(*e);
    return CASC_OK;
  };
  cudaEvent_t ev_in, ev_halo;
  if ((rc = new_event(&ev_in)) || (rc = new_event(&ev_halo))) return rc;
  // rank 0's halo rows stay zero (x_{-1} = 0); the others are overwritten by each exchange
  if (Hr > 0) {
    CASC_TRY(cudaMemsetAsync(w.Va, 0, (size_t)Hr * m * es, st));
    CASC_TRY(cudaMemsetAsync(w.Vb, 0, (size_t)Hr * m * es, st));
  }
  const size_t uhb = (size_t)uh * batch * p * es;     // bytes of the u halo
  CASC_TRY(cudaMemsetAsync(w.u_edge, 0, uhb, st));
  const int64_t Bu = boundary_rows(uh, batch, rows);
  CASC_TRY(cudaMemcpyAsync((char*)w.u_edge + uhb, u_loc, (size_t)Bu * p * es, cudaMemcpyDeviceToDevice, st));
  CASC_TRY(cudaEventRecord(ev_in, st));

  // ---- u halo: the last uh time rows of rank r-1's u (one contiguous block of uh * batch * p)
  {
    CASC_TRY(cudaStreamWaitEvent(cs, ev_in, 0));      // before the scope: it times the transfer only
    ProfScope ps(cs, K_SEQ_HALO, 2.0 * uhb, 0.0);
    if ((rc = exchange(c, (const char*)u_loc + (size_t)(rows - (int64_t)uh * batch) * p * es, uhb, w.u_edge, uhb,
                       nullptr, cs, ev_halo)))
      return rc;
  }
  const double dr = (double)rows;
  const int pipe = tf32 ? PIPE_TF32 : PIPE_BF16;
  const double xf = tf32 ? 3.0 : 1.0;
  auto two_launches = [&](MimoGemm g, MimoGemm gb, int64_t s_time, int cls, double bytes, double flops) -> int {
    // interior rows (every operand local) now; boundary rows once the halo has landed
    const int64_t Bs = boundary_rows(s_time, batch, rows);
    int r2;
    {
      ProfScope ps(st, cls, bytes * (dr - Bs) / dr, flops * (dr - Bs) / dr);
      ps.exec(bytes * (dr - Bs) / dr, xf * flops * (dr - Bs) / dr, pipe);
      if (Bs < rows && (r2 = step_gemm(g, rows, (int)(Bs / 128), tf32, st))) return r2;
    }
    CASC_TRY(cudaStreamWaitEvent(st, ev_halo, 0));
    ProfScope ps(st, cls, bytes * Bs / dr, flops * Bs / dr);
    ps.exec(bytes * Bs / dr, xf * flops * Bs / dr, pipe);
    return step_gemm(gb, Bs, 0, tf32, st);
  };

  if (Ne == 0) {                       // y = (C Bbar + D) u_l + (C Abar Bbar) u_{l-1}
    MimoGemm g{}, gb{};
    g.src[0] = {u_loc, w.mw.CBD, p, 0};
    g.src[1] = {u_loc, w.mw.CAB, p, batch};
    g.n_src = 2; g.out = y_loc; g.n_out = q;
    gb = g;
    gb.src[0] = {w.u_edge, w.mw.CBD, p, 0};
    gb.src[1] = {w.u_edge, w.mw.CAB, p, batch};
    gb.src[0].row0 = gb.src[1].row0 = uh * batch;
    return two_launches(g, gb, 1, K_MIMO_LAST, dr * (p + q) * es, dr * 4.0 * q * p);
  }
  // ---- first step: the Krylov head v^(2) = sum_{j<4} (Abar^j Bbar) u_{l-j} -> Vb for Ne >= 2 (R28),
  // else v^(1) = Bbar u_l + Abar Bbar u_{l-1} -> Va (local rows behind the halo)
  const int k0 = Ne >= 2 ? 2 : 1;
  {
    const void* Wj[4] = {w.mw.Bb, w.mw.AB, w.mw.A2B, w.mw.A3B};
    MimoGemm g{};
    g.n_src = Ne >= 2 ? 4 : 2;
    for (int j = 0; j < g.n_src; ++j) g.src[j] = {u_loc, Wj[j], p, (int64_t)j * batch};
    g.out = k0 == 2 ? w.Vb : w.Va; g.out_row0 = Hr; g.n_out = m;
    MimoGemm gb = g;
    for (int j = 0; j < g.n_src; ++j) {
      gb.src[j] = {w.u_edge, Wj[j], p, (int64_t)j * batch};
      gb.src[j].row0 = uh * batch;
    }
    if ((rc = two_launches(g, gb, uh, K_MIMO_FIRST, dr * (p + m) * es, dr * 2.0 * g.n_src * m * p))) return rc;
  }
  // ---- stages k = k0 .. kl-1 and the output step (from v^(kl), kl = Ne or Ne - 1 with the fold,
  // R31): before each, the halo of the rows of v^(k) it reads before l (2^k, or mimo_out_halo)
  const int kl = mimo_fold(Ne) ? Ne - 1 : Ne;
  for (int k = k0; k <= kl; ++k) {
    void* Vs = (k - 1) % 2 == 0 ? w.Va : w.Vb;       // holds v^(k)
    void* Vd = (k % 2 == 0) ? w.Va : w.Vb;
    const int64_t d_time = k < kl ? ((int64_t)1 << k) : mimo_out_halo(Ne);
    const int64_t d = d_time * batch;                // halo rows of this step
    cudaEvent_t ev_tail;
    if ((rc = new_event(&ev_tail))) return rc;
    CASC_TRY(cudaEventRecord(ev_tail, st));          // v^(k) complete on every local row
    {
      CASC_TRY(cudaStreamWaitEvent(cs, ev_tail, 0));
      ProfScope ps(cs, K_SEQ_HALO, 2.0 * d * m * es, 0.0);
      if ((rc = exchange(c, (const char*)Vs + (size_t)(Hr + rows - d) * m * es, (size_t)d * m * es,
                         (char*)Vs + (size_t)(Hr - d) * m * es, (size_t)d * m * es, nullptr, cs, ev_halo)))
        return rc;
    }
    MimoGemm g{};
    if (k < kl) {
      const void* Wk = tf32 ? static_cast<const void*>(P.f32 + k * 2 * mm) : static_cast<const void*>(P.b16 + k * mm);
      g.src[0] = {Vs, Wk, m, d};
      g.src[0].row0 = Hr;
      g.n_src = 1; g.R = Vs; g.R_row0 = Hr; g.out = Vd; g.out_row0 = Hr; g.n_out = m;
      if ((rc = two_launches(g, g, (int64_t)1 << k, K_MIMO_STAGE, dr * m * es * 2.0, dr * 2.0 * (double)mm))) return rc;
    } else {                           // y = C v + (C P_Ne) v_{l-2^Ne} + D u, or the folded form (R31)
      mimo_output_gemm(g, w.mw, Ne, m, p, q, Vs, Hr, u_loc, 0, D != nullptr, batch);
      g.out = y_loc; g.n_out = q;
      const double k_in = (double)(g.n_src - (D ? 1 : 0)) * m + (D ? p : 0);
      if ((rc = two_launches(g, g, d_time, K_MIMO_LAST, dr * (m + p + q) * es, dr * 2.0 * q * k_in)))
        return rc;
    }
  }
  return CASC_OK;
}

}  // extern "C"
