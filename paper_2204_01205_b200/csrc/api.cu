// libfno C ABI: plan / communicator / workspace logic on the host and the
// stream-ordered orchestration of the kernels and NCCL exchanges.
//
// Forward spectral convolution on P = px*py ranks:
//   pass A (t, z local; I_1)  -> exchange 1 (R_{P_xy -> P_kz})
//   -> pass B: y fwd, x fwd (I_2), mixing on owned kz, x inv, y inv
//   -> exchange 2 (R_{P_kz -> P_xy}, the adjoint) -> pass C (z, t inverse
//   fused with the DFNO block epilogue).
// Only the retained-mode slab travels: truncation happens before the exchange
// (reading Q9).
#include <cudaTypedefs.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/fno.h"
#include "launch.h"

using namespace fno;

namespace {

thread_local std::string g_err;

fno_status fail(fno_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define FNO_CUDA(call, stage)                                                                        \
  do {                                                                                               \
    cudaError_t _e = (call);                                                                         \
    if (_e != cudaSuccess) return fail(FNO_ERR_CUDA, std::string(stage) + ": " + cudaGetErrorString(_e)); \
  } while (0)
#define FNO_NCCL(call, stage)                                                                        \
  do {                                                                                               \
    ncclResult_t _r = (call);                                                                        \
    if (_r != ncclSuccess) return fail(FNO_ERR_NCCL, std::string(stage) + ": " + ncclGetErrorString(_r)); \
  } while (0)

void block_range(long long n, int p, int i, long long* lo, long long* hi) {
  long long q = n / p, r = n % p;
  *lo = i * q + std::min<long long>(i, r);
  *hi = *lo + q + (i < r ? 1 : 0);
}

// smallest L in the supported list that divides n and is >= need
template <class Pred>
int choose_L(long long n, long long need, Pred supported, const std::vector<int>& cands) {
  int best = 0;
  for (int L : cands)
    if (n % L == 0 && L >= need && supported(L) && (best == 0 || L < best)) best = L;
  return best;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

enum Stage { ST_PASS_A, ST_EX1, ST_B_YF, ST_B_XF, ST_MIX, ST_B_XI, ST_B_YI, ST_EX2, ST_PASS_C, ST_DWP, ST_DW, ST_N };
static const char* kStageNames[2 * ST_N] = {
    "fwd.pass_a", "fwd.exchange_1", "fwd.b_y_fwd", "fwd.b_x_fwd", "fwd.mix", "fwd.b_x_inv", "fwd.b_y_inv", "fwd.exchange_2", "fwd.pass_c", "fwd.unused_dw", "fwd.unused",
    "bwd.pass_a", "bwd.exchange_1", "bwd.b_y_fwd", "bwd.b_x_fwd", "bwd.mix", "bwd.b_x_inv", "bwd.b_y_inv", "bwd.exchange_2", "bwd.pass_c", "bwd.dw", "bwd.dw_reduce"};

static std::atomic<unsigned long long> g_launches{0};

struct Prof {
  bool on = false;
  std::vector<cudaEvent_t> ev;
  size_t used = 0;
  std::vector<std::pair<int, size_t>> recs;  // (stage, index of start event)
};

struct fno_comm_s {
  ncclComm_t nccl = nullptr;
  int nranks = 1, rank = 0;
};

struct fno_plan_s {
  fno_problem pb;
  fno_comm_t comm = nullptr;
  int P = 1, rank = 0, px = 1, py = 1, ix = 0, iy = 0;
  long long X, Y, Z, T, Xl, Yl;
  int B, C, mx, my, mz, mt;
  int act_gelu = 1;
  std::vector<int> kz_lo;  // P+1
  int nkz = 0;             // own block
  int LZ, LT, LX, LY;
  int Qz, Qt, Qx, Qy;
  int num_sms = 148;
  size_t smem_a[3] = {0, 0, 0};
  int np_a[3] = {1, 1, 1}, ns_a[3] = {2, 2, 2}, tma_a = 0, grid_a_m[3] = {1, 1, 1};
  // pass C kernel families per epilogue mode (EPI_U, EPI_FWD, EPI_BWD): index
  // family - 1 (1 generic pass_c, 2 pass_c2 FFMA, 3 pass_c3 tcgen05 1x1,
  // 4 pass_c4 warp-specialised tcgen05); cp == 0: not eligible
  struct KCfg {
    int cp = 0, tch = 0, vw = 1, nx = 0, grid = 1;
    size_t smem = 0;
  };
  KCfg kc[4][3];
  int fam[3] = {1, 1, 1};                      // the family each mode launches (fno_plan_set_pass_c)
  // family 5 (backward only): split backward, dv = W^T dz + S^T dz by the
  // forward-mode kernel of fam[EPI_FWD] (W^T, no bias, identity), dW / db by the
  // streaming dw_partial kernel (dw.cu) over dz and v; dw_grid CTAs, C <= 20
  int dw_grid = 0;
  long long mloc = 0;      // owned modes: 4 mx my nkz mt
  // workspace (bytes offsets)
  void* ws = nullptr;
  size_t ws_bytes = 0;
  size_t o_slab_xy, o_slab_kz, o_h, o_vhat, o_what, o_ghat, o_dwpart, o_dwall, o_dwloc, o_dz, o_bar, o_ipc, total;
  // peer exchange (fno_plan_connect_peers): every rank's workspace mapped over NVLink
  int peer = 0;
  int group = 0;                  // fno_group_connect: one of P plans of one process / device
  std::vector<char*> peer_ws;     // [P] workspace base of rank d in this process's address space
  std::vector<void*> ipc_opened;  // mappings to close at destroy
  size_t n_slab_xy, n_slab_kz, n_h, n_mode;
  int max_grid_c = 0;
  // caller-side partition of the fields (fno_plan_set_io_partition)
  int io[4] = {1, 1, 1, 1};
  bool io_on = false;
  size_t o_io_a = 0, o_io_b = 0, o_io_c = 0, o_io_ws = 0, io_ws_bytes = 0;
  int dir = 0;  // 0 forward call, 1 backward call (profiling labels)
  Prof prof;
  ~fno_plan_s() {
    for (cudaEvent_t e : prof.ev) cudaEventDestroy(e);
    for (void* m : ipc_opened) cudaIpcCloseMemHandle(m);
  }
};

namespace {
// records CUDA events around one stage on the launching stream when profiling
struct StageScope {
  fno_plan_t p;
  int stage;
  cudaStream_t st;
  size_t i0 = 0;
  bool on;
  size_t next() {
    if (p->prof.used == p->prof.ev.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      p->prof.ev.push_back(e);
    }
    return p->prof.used++;
  }
  StageScope(fno_plan_t p_, int s, cudaStream_t st_) : p(p_), stage(s), st(st_), on(p_->prof.on) {
    if (on) {
      i0 = next();
      next();
      cudaEventRecord(p->prof.ev[i0], st);
    }
  }
  ~StageScope() {
    if (on) {
      cudaEventRecord(p->prof.ev[i0 + 1], st);
      p->prof.recs.emplace_back(stage + p->dir * ST_N, i0);
    }
  }
};
}  // namespace

#define FNO_LAUNCH(p, stage, call, what) \
  do {                                   \
    StageScope _sc((p), (stage), st);    \
    FNO_CUDA(call, what);                \
    g_launches++;                        \
  } while (0)

// ---------------------------------------------------------------------------
// status / version
// ---------------------------------------------------------------------------
extern "C" const char* fno_status_string(fno_status s) {
  switch (s) {
    case FNO_OK: return "FNO_OK";
    case FNO_ERR_INVALID_ARGUMENT: return "FNO_ERR_INVALID_ARGUMENT";
    case FNO_ERR_PLAN: return "FNO_ERR_PLAN";
    case FNO_ERR_INVALID_STATE: return "FNO_ERR_INVALID_STATE";
    case FNO_ERR_CUDA: return "FNO_ERR_CUDA";
    case FNO_ERR_NCCL: return "FNO_ERR_NCCL";
    case FNO_ERR_WORKSPACE: return "FNO_ERR_WORKSPACE";
  }
  return "FNO_ERR_UNKNOWN";
}
extern "C" const char* fno_last_error(void) { return g_err.c_str(); }
extern "C" int fno_abi_version(void) { return FNO_ABI_VERSION; }

// ---------------------------------------------------------------------------
// communicator
// ---------------------------------------------------------------------------
extern "C" fno_status fno_comm_unique_id(uint8_t id[128]) {
  if (!id) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_comm_unique_id: id is NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId u;
  FNO_NCCL(ncclGetUniqueId(&u), "ncclGetUniqueId");
  std::memcpy(id, &u, 128);
  return FNO_OK;
}

extern "C" fno_status fno_comm_init(const uint8_t id[128], int nranks, int rank, fno_comm_t* comm) {
  if (!id || !comm || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(FNO_ERR_INVALID_ARGUMENT, "fno_comm_init: bad arguments");
  auto* c = new fno_comm_s();
  c->nranks = nranks;
  c->rank = rank;
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(FNO_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  }
  *comm = c;
  return FNO_OK;
}

extern "C" fno_status fno_comm_init_local(int nranks, int rank, fno_comm_t* comm) {
  if (!comm || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(FNO_ERR_INVALID_ARGUMENT, "fno_comm_init_local: bad arguments");
  auto* c = new fno_comm_s();
  c->nranks = nranks;
  c->rank = rank;
  *comm = c;
  return FNO_OK;
}

extern "C" fno_status fno_comm_destroy(fno_comm_t comm) {
  if (!comm) return FNO_OK;
  if (comm->nccl) ncclCommDestroy(comm->nccl);
  delete comm;
  return FNO_OK;
}

extern "C" fno_status fno_comm_size(fno_comm_t comm, int* nranks, int* rank) {
  if (!comm || !nranks || !rank) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_comm_size: NULL argument");
  *nranks = comm->nranks;
  *rank = comm->rank;
  return FNO_OK;
}

// ---------------------------------------------------------------------------
// plan
// ---------------------------------------------------------------------------
extern "C" fno_status fno_plan_create(const fno_problem* pb, fno_comm_t comm, fno_plan_t* out) {
  if (!pb || !out) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_plan_create: NULL argument");
  for (int d = 0; d < 4; ++d)
    if (pb->grid[d] <= 0) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_plan_create: grid extents must be > 0");
  if (pb->batch < 1 || pb->width < 1) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_plan_create: batch and width must be >= 1");
  for (int d = 0; d < 3; ++d)
    if (pb->modes[d] < 1 || 2LL * pb->modes[d] > pb->grid[d])
      return fail(FNO_ERR_INVALID_ARGUMENT, "fno_plan_create: spatial modes need 1 <= m and 2m <= n (P:52, reading Q2)");
  if (pb->modes[3] < 1 || pb->modes[3] > pb->grid[3] / 2 + 1)
    return fail(FNO_ERR_INVALID_ARGUMENT, "fno_plan_create: time modes need 1 <= mt <= T/2+1 (reading Q2)");
  if (pb->pgrid[0] < 1 || pb->pgrid[1] < 1) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_plan_create: pgrid entries must be >= 1");
  if (pb->flags & ~1u) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_plan_create: unknown flags");
  const int P = pb->pgrid[0] * pb->pgrid[1];
  if (P > FNO_MAXP) return fail(FNO_ERR_PLAN, "fno_plan_create: more than 64 ranks");
  int nranks = 1, rank = 0;
  if (comm) { nranks = comm->nranks; rank = comm->rank; }
  if (nranks != P) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_plan_create: px*py must equal the communicator size (NULL comm => 1)");
  if (pb->grid[0] % pb->pgrid[0] || pb->grid[1] % pb->pgrid[1])
    return fail(FNO_ERR_INVALID_ARGUMENT, "fno_plan_create: X % px and Y % py must be 0 (balanced uneven boxes are not supported yet)");
  if (2 * pb->modes[2] > 32767) return fail(FNO_ERR_PLAN, "fno_plan_create: too many z modes");
  if (pb->grid[3] > 512 || pb->grid[2] > 4096) return fail(FNO_ERR_PLAN, "fno_plan_create: T > 512 or Z > 4096 not supported");

  auto* p = new fno_plan_s();
  p->pb = *pb;
  p->comm = comm;
  p->P = P;
  p->rank = rank;
  p->px = pb->pgrid[0];
  p->py = pb->pgrid[1];
  p->ix = rank / p->py;
  p->iy = rank % p->py;
  p->X = pb->grid[0]; p->Y = pb->grid[1]; p->Z = pb->grid[2]; p->T = pb->grid[3];
  p->Xl = p->X / p->px; p->Yl = p->Y / p->py;
  p->io[0] = p->px; p->io[1] = p->py; p->io[2] = 1; p->io[3] = 1;   // the caller's partition is the plan's until set
  p->B = pb->batch; p->C = pb->width;
  p->mx = pb->modes[0]; p->my = pb->modes[1]; p->mz = pb->modes[2]; p->mt = pb->modes[3];
  p->act_gelu = (pb->flags & FNO_ACT_NONE) ? 0 : 1;
  p->kz_lo.resize(P + 1);
  for (int d = 0; d < P; ++d) {
    long long lo, hi;
    block_range(2LL * p->mz, P, d, &lo, &hi);
    p->kz_lo[d] = int(lo);
    p->kz_lo[d + 1] = int(hi);
  }
  p->nkz = p->kz_lo[rank + 1] - p->kz_lo[rank];

  // transform sizes (readings: z real input needs kz' = 0..mz; t needs
  // min(2mt-1, T) residues; x, y need 2m residues)
  const std::vector<int> ac_z = {2, 4, 8, 16, 32};
  const std::vector<int> ac_t = {4, 5, 8, 15, 16, 30, 32};
  const std::vector<int> bs = {2, 4, 5, 6, 8, 16, 30, 32};
  const long long need_t = std::min<long long>(2LL * p->mt - 1, p->T);
  p->LZ = 0; p->LT = 0;
  for (int lz : ac_z) {
    if (p->Z % lz || lz < p->mz + 1) continue;
    for (int lt : ac_t) {
      if (p->T % lt || lt < need_t || !ac_pair_supported(lz, lt)) continue;
      if (p->LZ == 0 || lz < p->LZ || (lz == p->LZ && lt < p->LT)) { p->LZ = lz; p->LT = lt; }
    }
  }
  p->LX = choose_L(p->X, 2LL * p->mx, b_size_supported, bs);
  p->LY = choose_L(p->Y, 2LL * p->my, b_size_supported, bs);
  if (!p->LZ || !p->LT || !p->LX || !p->LY) {
    char buf[256];
    std::snprintf(buf, sizeof buf, "fno_plan_create: no instantiated register-FFT size for grid (%lld,%lld,%lld,%lld) modes (%d,%d,%d,%d)",
                  p->X, p->Y, p->Z, p->T, p->mx, p->my, p->mz, p->mt);
    delete p;
    return fail(FNO_ERR_PLAN, buf);
  }
  p->Qz = int(p->Z / p->LZ); p->Qt = int(p->T / p->LT);
  p->Qx = int(p->X / p->LX); p->Qy = int(p->Y / p->LY);

  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && sms > 0) p->num_sms = sms;
  } else {
    cudaGetLastError();
  }

  // pass A batching (planes per TMA batch) per input mode
  for (int m = 0; m < 3; ++m) pass_a_config(int(p->Z), int(p->T), p->mz, m, &p->np_a[m], &p->ns_a[m], &p->smem_a[m], &p->tma_a);
  // pass C kernel families eligible for each epilogue mode
  for (int m = 0; m < 3; ++m) {
    fno_plan_s::KCfg& g = p->kc[0][m];
    g.cp = p->C;
    pass_c_config(p->C, int(p->Z), int(p->T), p->mz, p->mt, p->LZ, m, &g.tch, &g.vw, &g.smem);
    int cp, tch, vw, nx, ns;
    size_t sm;
    if (m != EPI_U && pass_c2_config(p->C, int(p->Z), int(p->T), p->mz, p->mt, p->LZ, m, &cp, &tch, &vw, &sm, &nx)) {
      fno_plan_s::KCfg& h = p->kc[1][m];
      h.cp = cp; h.tch = tch; h.vw = vw; h.smem = sm; h.nx = nx;
    }
    if (m == EPI_FWD && pass_c3_config(p->C, int(p->Z), int(p->T), p->mz, p->mt, p->LZ, m, &cp, &tch, &sm)) {
      fno_plan_s::KCfg& h = p->kc[2][m];
      h.cp = cp; h.tch = tch; h.smem = sm;
    }
    if (pass_c4_config(p->C, int(p->Z), int(p->T), p->mz, p->mt, p->LZ, m, &cp, &ns, &sm)) {
      fno_plan_s::KCfg& h = p->kc[3][m];
      h.cp = cp; h.tch = 128 / p->LZ; h.nx = ns; h.smem = sm;
    }
  }
  // default choice, by measurement on B200 (profiles/r02/ab_pass_c.md, after the
  // pass_c4 code-size cut): the spectral u path and the layer forward on pass_c4
  // (c2 0.945 vs 0.960 ms per layer forward with pass_c3, c4 3.99 vs 4.11 with
  // pass_c2); the layer backward split (family 5: dv by the forward kernel, dW / db
  // by dw_partial; c2 1.29 vs 1.31, c3 1.94 vs 2.08, c4 5.50 vs 5.58 ms per layer
  // backward against the fused FFMA pass_c2; the tcgen05 pass_c4 backward, 2.05 ms
  // at c2, serialises its three operand splits)
  auto ok = [&](int f, int m) { return f == 5 ? (m == EPI_BWD && p->C <= 20) : p->kc[f - 1][m].cp > 0; };
  p->fam[EPI_U] = ok(4, EPI_U) ? 4 : 1;
  p->fam[EPI_FWD] = ok(4, EPI_FWD) ? 4 : ok(3, EPI_FWD) ? 3 : ok(2, EPI_FWD) ? 2 : 1;
  p->fam[EPI_BWD] = ok(5, EPI_BWD) ? 5 : ok(2, EPI_BWD) ? 2 : ok(4, EPI_BWD) ? 4 : 1;
#ifdef FNO_DEV_KNOBS   // development builds only: FNO_PASS_C_FAM=<u><fwd><bwd> digits force families
  if (const char* fe = std::getenv("FNO_PASS_C_FAM")) {
    for (int m = 0; m < 3 && fe[m]; ++m) {
      const int f = fe[m] - '0';
      if (f >= 1 && f <= 5 && ok(f, m)) p->fam[m] = f;
    }
  }
#endif
  const size_t smem_max = 227 * 1024;
  if (p->smem_a[MODE_DZ_GELU] > smem_max || p->kc[0][EPI_BWD].smem > smem_max) {
    char buf[200];
    std::snprintf(buf, sizeof buf, "fno_plan_create: shared memory per CTA too large (pass A %zu, pass C %zu bytes)",
                  p->smem_a[MODE_DZ_GELU], p->kc[0][EPI_BWD].smem);
    delete p;
    return fail(FNO_ERR_PLAN, buf);
  }
  const long long n_planes = (long long)p->B * p->C * p->Xl * p->Yl;
  for (int m = 0; m < 3; ++m) {
    const long long n_batches = (n_planes + p->np_a[m] - 1) / p->np_a[m];
    const int per_sm_a = std::max(1, int(std::min<size_t>(pass_a_max_blocks(m, int(p->T)), (228 * 1024) / (p->smem_a[m] + 1024))));
    p->grid_a_m[m] = int(std::max<long long>(1, std::min<long long>(n_batches, (long long)p->num_sms * per_sm_a)));
  }
  const long long n_cols = (long long)p->B * p->Xl * p->Yl;
  auto grid_for = [&](size_t smem) {
    const int per_sm = std::max(1, int(std::min<size_t>(8, (228 * 1024) / (smem + 1024))));
    return int(std::max<long long>(1, std::min<long long>(n_cols, (long long)p->num_sms * per_sm)));
  };
  p->max_grid_c = 1;
  if (p->C <= 20) {
    p->dw_grid = dw_partial_grid(p->B, p->Xl * p->Yl * p->Z * p->T, p->num_sms);
    p->max_grid_c = std::max(p->max_grid_c, p->dw_grid);
  }
  for (int f = 0; f < 4; ++f)
    for (int m = 0; m < 3; ++m) {
      fno_plan_s::KCfg& g = p->kc[f][m];
      g.grid = f == 3 ? int(std::max<long long>(1, std::min<long long>(n_cols, p->num_sms)))   // one CTA per SM
                      : grid_for(g.smem);
      if (g.cp > 0) p->max_grid_c = std::max(p->max_grid_c, g.grid);
    }

  // workspace layout
  p->mloc = 4LL * p->mx * p->my * p->nkz * p->mt;
  p->n_slab_xy = size_t(p->B) * p->Xl * p->Yl * p->C * 2 * p->mz * p->mt;
  p->n_slab_kz = size_t(P) * p->B * p->Xl * p->Yl * p->C * p->nkz * p->mt;
  p->n_h = size_t(p->B) * p->nkz * p->C * p->X * 2 * p->my * p->mt;
  p->n_mode = size_t(p->B) * p->C * p->mloc;
  const size_t dwlen = size_t(p->C) * p->C + p->C;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += align256(bytes); return o; };
  // the peer-exchange barrier rows first: ranks write into each other's rows at
  // their OWN offset, so it must not depend on rank-specific sizes (nkz)
  p->o_bar = take(1024);                     // flag row [64] + epoch (zeroed at connect)
  p->o_slab_xy = take(p->n_slab_xy * 8);
  p->o_slab_kz = (P == 1) ? p->o_slab_xy : take(p->n_slab_kz * 8);
  p->o_h = take(p->n_h * 8);
  p->o_vhat = take(p->n_mode * 8);
  p->o_what = take(p->n_mode * 8);
  p->o_ghat = take(p->n_mode * 8);
  p->o_dwpart = take(size_t(p->max_grid_c) * dwlen * 4);
  p->o_dwloc = take(dwlen * 4);
  p->o_dwall = take(size_t(P) * dwlen * 4);
  p->o_dz = take(size_t(p->B) * p->C * p->Xl * p->Yl * p->Z * p->T * 4);   // dz = dy * sigma'(z) (bwd)
  p->o_ipc = take(size_t(P) * 256);          // peer-exchange handle all-gather
  p->total = off;
  *out = p;
  return FNO_OK;
}

extern "C" fno_status fno_plan_destroy(fno_plan_t p) {
  delete p;
  return FNO_OK;
}

extern "C" fno_status fno_plan_workspace_size(fno_plan_t p, size_t* bytes) {
  if (!p || !bytes) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_plan_workspace_size: NULL argument");
  *bytes = p->total;
  return FNO_OK;
}

extern "C" fno_status fno_plan_set_workspace(fno_plan_t p, void* dptr, size_t bytes) {
  if (!p) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_plan_set_workspace: NULL plan");
  if (!dptr || bytes < p->total) return fail(FNO_ERR_WORKSPACE, "fno_plan_set_workspace: workspace NULL or smaller than fno_plan_workspace_size");
  if (reinterpret_cast<uintptr_t>(dptr) & 255) return fail(FNO_ERR_WORKSPACE, "fno_plan_set_workspace: workspace must be 256-byte aligned");
  // the peers hold mappings of the current workspace (fno_plan_connect_peers)
  if (p->peer) return fail(FNO_ERR_INVALID_STATE, "fno_plan_set_workspace: peers are connected to the current workspace");
  p->ws = dptr;
  p->ws_bytes = bytes;
  return FNO_OK;
}

// Collective: map every rank's workspace into this process (CUDA IPC over
// NVLink) so pass A and the y-inverse store their exchange chunks straight
// into the owners' receive buffers.  No-op for P == 1.
extern "C" fno_status fno_plan_connect_peers(fno_plan_t p, void* stream) {
  if (!p) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_plan_connect_peers: NULL plan");
  if (p->P == 1) return FNO_OK;
  if (!p->ws) return fail(FNO_ERR_INVALID_STATE, "fno_plan_connect_peers: workspace not set");
  if (!p->comm || !p->comm->nccl) return fail(FNO_ERR_INVALID_STATE, "fno_plan_connect_peers: communicator missing");
  if (p->peer) return FNO_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  static PFN_cuMemGetAddressRange_v3020 range = nullptr;
  if (!range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      range = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(fn);
    else
      cudaGetLastError();
  }
  // Every rank contributes a record even when it cannot export its workspace
  // (no driver entry point, an allocator whose memory CUDA IPC refuses, ...),
  // so the all-gather below never leaves a rank behind; whether peer stores
  // are used is then decided collectively (all ranks or none).  Peer access is
  // not pre-checked with device ordinals (those are process-local, e.g. every
  // rank sees device 0 under per-rank CUDA_VISIBLE_DEVICES):
  // cudaIpcOpenMemHandle itself decides.
  struct Rec {
    cudaIpcMemHandle_t h;
    unsigned long long off;
    int ok;
  };
  static_assert(sizeof(Rec) <= 256, "handle record");
  Rec mine{};
  CUdeviceptr base = 0;
  size_t alloc = 0;
  if (range && range(&base, &alloc, reinterpret_cast<CUdeviceptr>(p->ws)) == CUDA_SUCCESS &&
      cudaIpcGetMemHandle(&mine.h, reinterpret_cast<void*>(base)) == cudaSuccess) {
    mine.off = reinterpret_cast<CUdeviceptr>(p->ws) - base;
    mine.ok = 1;
  } else {
    cudaGetLastError();
  }
  unsigned char* dbuf = static_cast<unsigned char*>(p->ws) + p->o_ipc;
  // barrier flag rows start at epoch 0 on every rank before any rank can write
  // into a peer's row (the handle all-gather below orders the two)
  FNO_CUDA(cudaMemsetAsync(static_cast<char*>(p->ws) + p->o_bar, 0, 1024, st), "peer barrier flags");
  FNO_CUDA(cudaMemcpyAsync(dbuf + size_t(p->rank) * 256, &mine, sizeof mine, cudaMemcpyHostToDevice, st), "ipc h2d");
  FNO_NCCL(ncclAllGather(dbuf + size_t(p->rank) * 256, dbuf, 256, ncclUint8, p->comm->nccl, st), "ipc all-gather");
  std::vector<unsigned char> all(size_t(p->P) * 256);
  FNO_CUDA(cudaMemcpyAsync(all.data(), dbuf, all.size(), cudaMemcpyDeviceToHost, st), "ipc d2h");
  FNO_CUDA(cudaStreamSynchronize(st), "fno_plan_connect_peers: sync");
  std::vector<char*> bases(p->P, nullptr);
  std::vector<void*> opened;
  int ok = 1;
  for (int d = 0; d < p->P && ok; ++d) {
    Rec r;
    std::memcpy(&r, all.data() + size_t(d) * 256, sizeof r);
    if (!r.ok) { ok = 0; break; }
    if (d == p->rank) {
      bases[d] = static_cast<char*>(p->ws);
      continue;
    }
    void* m = nullptr;
    if (cudaIpcOpenMemHandle(&m, r.h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      ok = 0;
      break;
    }
    opened.push_back(m);
    bases[d] = static_cast<char*>(m) + r.off;
  }
  // collective decision: peer stores only if every rank mapped every peer
  int* flag = reinterpret_cast<int*>(dbuf + size_t(p->rank) * 256);
  FNO_CUDA(cudaMemcpyAsync(flag, &ok, sizeof ok, cudaMemcpyHostToDevice, st), "peer flag h2d");
  FNO_NCCL(ncclAllReduce(flag, flag, 1, ncclInt, ncclMin, p->comm->nccl, st), "peer flag all-reduce");
  int all_ok = 0;
  FNO_CUDA(cudaMemcpyAsync(&all_ok, flag, sizeof all_ok, cudaMemcpyDeviceToHost, st), "peer flag d2h");
  FNO_CUDA(cudaStreamSynchronize(st), "fno_plan_connect_peers: sync");
  if (!all_ok) {   // every rank keeps the NCCL send/recv exchanges
    for (void* m : opened) cudaIpcCloseMemHandle(m);
    return FNO_OK;
  }
  p->ipc_opened.insert(p->ipc_opened.end(), opened.begin(), opened.end());
  p->peer_ws = bases;
  p->peer = 1;
  return FNO_OK;
}

extern "C" fno_status fno_plan_peer_enabled(fno_plan_t p, int* enabled) {
  if (!p || !enabled) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_plan_peer_enabled: NULL argument");
  *enabled = p->peer;
  return FNO_OK;
}

extern "C" fno_status fno_plan_pass_c_info(fno_plan_t p, int mode, int64_t info[4]) {
  if (!p || !info || mode < 0 || mode > 2) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_plan_pass_c_info: bad arguments");
  const int m = mode == 0 ? EPI_U : (mode == 1 ? EPI_FWD : EPI_BWD);
  const int f = p->fam[m];
  // family 5: the configuration of its dv kernel (the forward family's)
  const auto& g = f == 5 ? p->kc[p->fam[EPI_FWD] - 1][EPI_FWD] : p->kc[f - 1][m];
  info[0] = f; info[1] = g.cp; info[2] = g.nx; info[3] = int64_t(g.smem);
  return FNO_OK;
}

extern "C" fno_status fno_plan_set_pass_c(fno_plan_t p, int mode, int family) {
  if (!p || mode < 0 || mode > 2 || family < 1 || family > 5)
    return fail(FNO_ERR_INVALID_ARGUMENT, "fno_plan_set_pass_c: mode 0..2, family 1..5");
  const int m = mode == 0 ? EPI_U : (mode == 1 ? EPI_FWD : EPI_BWD);
  if (family == 5 ? (m != EPI_BWD || p->dw_grid == 0) : p->kc[family - 1][m].cp == 0)
    return fail(FNO_ERR_PLAN, "fno_plan_set_pass_c: that pass C kernel family does not cover this problem");
  p->fam[m] = family;
  return FNO_OK;
}

#ifdef FNO_C4_PROFILE
// development builds: the pass_c4 role timers of the last pass C launch ([grid][16] u64 in the pass B scratch H)
extern "C" fno_status fno_debug_c4_timers(fno_plan_t p, unsigned long long* host, int n) {
  if (!p || !host || !p->ws) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_debug_c4_timers");
  FNO_CUDA(cudaMemcpy(host, static_cast<char*>(p->ws) + p->o_h, size_t(n) * 8, cudaMemcpyDeviceToHost), "timers");
  return FNO_OK;
}
#endif

extern "C" fno_status fno_plan_local_box(fno_plan_t p, int64_t lo[4], int64_t hi[4]) {
  if (!p || !lo || !hi) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_plan_local_box: NULL argument");
  lo[0] = p->ix * p->Xl; hi[0] = lo[0] + p->Xl;
  lo[1] = p->iy * p->Yl; hi[1] = lo[1] + p->Yl;
  lo[2] = 0; hi[2] = p->Z;
  lo[3] = 0; hi[3] = p->T;
  return FNO_OK;
}

extern "C" fno_status fno_plan_owned_modes(fno_plan_t p, int32_t* kz_lo, int32_t* kz_hi) {
  if (!p || !kz_lo || !kz_hi) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_plan_owned_modes: NULL argument");
  *kz_lo = p->kz_lo[p->rank];
  *kz_hi = p->kz_lo[p->rank + 1];
  return FNO_OK;
}

extern "C" fno_status fno_plan_profile_enable(fno_plan_t p, int enable) {
  if (!p) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_plan_profile_enable: NULL plan");
  p->prof.on = enable != 0;
  return FNO_OK;
}

extern "C" fno_status fno_plan_profile_read(fno_plan_t p, double* ms, int64_t* count, int nstages) {
  if (!p || !ms || !count || nstages < 2 * ST_N) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_plan_profile_read: bad arguments");
  for (int i = 0; i < nstages; ++i) { ms[i] = 0.0; count[i] = 0; }
  for (auto& r : p->prof.recs) {
    float t = 0.f;
    FNO_CUDA(cudaEventSynchronize(p->prof.ev[r.second + 1]), "fno_plan_profile_read");
    FNO_CUDA(cudaEventElapsedTime(&t, p->prof.ev[r.second], p->prof.ev[r.second + 1]), "fno_plan_profile_read");
    ms[r.first] += t;
    count[r.first] += 1;
  }
  p->prof.recs.clear();
  p->prof.used = 0;
  return FNO_OK;
}

extern "C" int fno_profile_stage_count(void) { return 2 * ST_N; }
extern "C" const char* fno_profile_stage_name(int i) { return (i >= 0 && i < 2 * ST_N) ? kStageNames[i] : ""; }
extern "C" unsigned long long fno_kernel_launches(void) { return g_launches.load(); }

extern "C" fno_status fno_plan_vhat_elems(fno_plan_t p, size_t* elems) {
  if (!p || !elems) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_plan_vhat_elems: NULL argument");
  *elems = p->n_mode;
  return FNO_OK;
}

// ---------------------------------------------------------------------------
// orchestration
// ---------------------------------------------------------------------------
namespace {

template <class T>
T* wsp(fno_plan_t p, size_t off) {
  return reinterpret_cast<T*>(static_cast<char*>(p->ws) + off);
}

KzSlab make_kzslab(fno_plan_t p) {
  KzSlab s{};
  s.P = p->P;
  long long off = 0;
  const long long per = (long long)p->B * p->Xl * p->Yl * p->C * p->mt;
  for (int d = 0; d <= p->P; ++d) s.kz_lo[d] = p->kz_lo[d];
  for (int d = 0; d < p->P; ++d) {
    s.off[d] = off;
    off += per * (p->kz_lo[d + 1] - p->kz_lo[d]);
  }
  // pass A destinations: local send buffer, or this rank's block [src = rank] of
  // owner d's kz-ordered receive buffer (chunks of per * nkz_d)
  for (int d = 0; d < p->P; ++d) {
    const long long nkz_d = p->kz_lo[d + 1] - p->kz_lo[d];
    if (p->peer)
      s.dst[d] = reinterpret_cast<float2*>(p->peer_ws[d] + p->o_slab_kz) + (long long)p->rank * per * nkz_d;
    else if (p->ws)
      s.dst[d] = wsp<float2>(p, p->o_slab_xy) + s.off[d];
  }
  return s;
}

PassBParams make_b(fno_plan_t p, const float2* in, float2* out, int Q) {
  PassBParams b{};
  b.in = in; b.out = out;
  b.B = p->B; b.C = p->C; b.X = int(p->X); b.Y = int(p->Y); b.Xl = int(p->Xl); b.Yl = int(p->Yl);
  b.py = p->py; b.nkz = p->nkz; b.mt = p->mt; b.mx = p->mx; b.my = p->my; b.Q = Q;
  b.chunk = (long long)p->B * p->Xl * p->Yl * p->C * p->nkz * p->mt;
  return b;
}

// exchange 1 (forward): kz-owner ordered send buffer -> x/y-source ordered receive buffer
// peer exchange: the data already went over NVLink inside pass A / the
// y-inverse; the exchange is a barrier (one-int NCCL all-reduce), after which
// every rank's receive buffer is complete (writers fenced at system scope)
fno_status peer_barrier(fno_plan_t p, int stage, const char* what, cudaStream_t st) {
  // flag rows at o_bar: [0, 64) flags (u64 per source rank), [64] the epoch
  PeerBarrierParams b{};
  b.P = p->P;
  b.rank = p->rank;
  b.my_flags = wsp<unsigned long long>(p, p->o_bar);
  b.epoch = b.my_flags + FNO_MAXP;
  for (int d = 0; d < p->P; ++d) b.peer_flags[d] = reinterpret_cast<unsigned long long*>(p->peer_ws[d] + p->o_bar);
  FNO_LAUNCH(p, stage, launch_peer_barrier(b, st), what);
  return FNO_OK;
}

fno_status exchange_fwd(fno_plan_t p, cudaStream_t st) {
  if (p->P == 1 || p->group) return FNO_OK;   // group: stream order is the barrier
  if (p->peer) return peer_barrier(p, ST_EX1, "exchange 1 (peer barrier)", st);
  const KzSlab s = make_kzslab(p);
  const size_t per = size_t(p->B) * p->Xl * p->Yl * p->C * p->mt;  // complex per kz plane
  float2* send = wsp<float2>(p, p->o_slab_xy);
  float2* recv = wsp<float2>(p, p->o_slab_kz);
  StageScope sc(p, ST_EX1, st);
  FNO_NCCL(ncclGroupStart(), "exchange 1: ncclGroupStart");
  for (int d = 0; d < p->P; ++d) {
    const size_t ns = per * (p->kz_lo[d + 1] - p->kz_lo[d]);
    const size_t nr = per * p->nkz;
    if (ns) FNO_NCCL(ncclSend(send + s.off[d], 2 * ns, ncclFloat, d, p->comm->nccl, st), "exchange 1: ncclSend");
    if (nr) FNO_NCCL(ncclRecv(recv + d * nr, 2 * nr, ncclFloat, d, p->comm->nccl, st), "exchange 1: ncclRecv");
  }
  FNO_NCCL(ncclGroupEnd(), "exchange 1: ncclGroupEnd");
  return FNO_OK;
}

// exchange 2 (adjoint): x/y-destination ordered -> kz-owner ordered
fno_status exchange_bwd(fno_plan_t p, cudaStream_t st) {
  if (p->P == 1 || p->group) return FNO_OK;
  if (p->peer) return peer_barrier(p, ST_EX2, "exchange 2 (peer barrier)", st);
  const KzSlab s = make_kzslab(p);
  const size_t per = size_t(p->B) * p->Xl * p->Yl * p->C * p->mt;
  float2* send = wsp<float2>(p, p->o_slab_kz);
  float2* recv = wsp<float2>(p, p->o_slab_xy);
  StageScope sc(p, ST_EX2, st);
  FNO_NCCL(ncclGroupStart(), "exchange 2: ncclGroupStart");
  for (int d = 0; d < p->P; ++d) {
    const size_t ns = per * p->nkz;
    const size_t nr = per * (p->kz_lo[d + 1] - p->kz_lo[d]);
    if (ns) FNO_NCCL(ncclSend(send + d * ns, 2 * ns, ncclFloat, d, p->comm->nccl, st), "exchange 2: ncclSend");
    if (nr) FNO_NCCL(ncclRecv(recv + s.off[d], 2 * nr, ncclFloat, d, p->comm->nccl, st), "exchange 2: ncclRecv");
  }
  FNO_NCCL(ncclGroupEnd(), "exchange 2: ncclGroupEnd");
  return FNO_OK;
}

fno_status run_pass_a(fno_plan_t p, const float* in0, const float* in1, int mode, cudaStream_t st) {
  PassAParams a{};
  a.in0 = in0; a.in1 = in1;
  a.out = wsp<float2>(p, p->o_slab_xy);
  a.n_planes = (long long)p->B * p->C * p->Xl * p->Yl;
  a.Z = int(p->Z); a.T = int(p->T); a.mz = p->mz; a.mt = p->mt; a.Qz = p->Qz; a.Qt = p->Qt; a.NP = p->np_a[mode]; a.NS = p->ns_a[mode];
  a.C = p->C; a.Xl = int(p->Xl); a.Yl = int(p->Yl);
  a.use_tma = p->tma_a;
  a.dz_out = wsp<float>(p, p->o_dz);
  a.slab = make_kzslab(p);
  a.peer = p->peer;
  FNO_LAUNCH(p, ST_PASS_A, launch_pass_a(a, p->LZ, p->LT, mode, p->grid_a_m[mode], p->smem_a[mode], st), "pass A");
  return FNO_OK;
}

// pass B forward half: slab (kz block, x/y-source ordered) -> V^ (owned modes)
fno_status run_b_fwd(fno_plan_t p, float2* vhat_out, cudaStream_t st) {
  if (p->nkz == 0) return FNO_OK;
  float2* slab = wsp<float2>(p, p->o_slab_kz);
  float2* H = wsp<float2>(p, p->o_h);
  FNO_LAUNCH(p, ST_B_YF, launch_b_yfwd(make_b(p, slab, H, p->Qy), p->LY, st), "pass B y-forward");
  FNO_LAUNCH(p, ST_B_XF, launch_b_xfwd(make_b(p, H, vhat_out, p->Qx), p->LX, st), "pass B x-forward");
  return FNO_OK;
}

// pass B inverse half: W^ -> slab (x/y-destination ordered)
fno_status run_b_inv(fno_plan_t p, const float2* what, cudaStream_t st) {
  if (p->nkz == 0) return FNO_OK;
  float2* slab = wsp<float2>(p, p->o_slab_kz);
  float2* H = wsp<float2>(p, p->o_h);
  FNO_LAUNCH(p, ST_B_XI, launch_b_xinv(make_b(p, what, H, p->Qx), p->LX, st), "pass B x-inverse");
  PassBParams yb = make_b(p, H, slab, p->Qy);
  // destinations of the y-inverse: local send buffer chunks [d], or this rank's
  // block [owner = rank] of rank d's x/y-ordered receive buffer
  const KzSlab ks = make_kzslab(p);
  yb.P = p->P;
  yb.peer = p->peer;
  for (int d = 0; d < p->P; ++d)
    yb.dst[d] = p->peer ? reinterpret_cast<float2*>(p->peer_ws[d] + p->o_slab_xy) + ks.off[p->rank] : slab + d * yb.chunk;
  FNO_LAUNCH(p, ST_B_YI, launch_b_yinv(yb, p->LY, st), "pass B y-inverse");
  return FNO_OK;
}

MixParams make_mix(fno_plan_t p) {
  MixParams m{};
  m.M = p->mloc; m.B = p->B; m.C = p->C; m.mt = p->mt; m.T = int(p->T);
  m.inv_n = float(1.0 / (double(p->X) * p->Y * p->Z * p->T));
  return m;
}

PassCParams make_c(fno_plan_t p, int mode) {
  PassCParams c{};
#ifdef FNO_ABLATE_BUILD
  {
    static const int ablate = [] { const char* e = std::getenv("FNO_ABLATE"); return e ? std::atoi(e) : 0; }();
    c.ablate = ablate;
  }
#endif
  c.in = wsp<float2>(p, p->o_slab_xy);
  c.dWpart = wsp<float>(p, p->o_dwpart);   // bwd: dW / db partial rows
#ifdef FNO_C4_PROFILE
  c.prof = wsp<unsigned long long>(p, p->o_h);   // development builds: pass_c4 role timers
#endif
  c.n_cols = (long long)p->B * p->Xl * p->Yl;
  c.B = p->B; c.C = p->C; c.Xl = int(p->Xl); c.Yl = int(p->Yl); c.Z = int(p->Z); c.T = int(p->T);
  c.mz = p->mz; c.mt = p->mt; c.Qz = p->Qz; c.Qt = p->Qt;
  c.act_gelu = p->act_gelu;
  c.inv_n = float(1.0 / (double(p->X) * p->Y * p->Z * p->T));
  c.slab = make_kzslab(p);
  return c;
}

// the selected pass C kernel for the mode (p->fam); *grid_used: its CTA count
// (the number of dW / db partial rows of the backward).  pass_c4 falls back to
// the next eligible family when the tensors' alignment rules out its TMA view.
cudaError_t run_pass_c(fno_plan_t p, const PassCParams& c0, int mode, cudaStream_t st, int* grid_used = nullptr) {
  int f = p->fam[mode];
  for (;;) {
    const auto& g = p->kc[f - 1][mode];
    PassCParams c = c0;
    c.TCH = g.tch;
    c.VW = g.vw;
    c.NX = g.nx;
    if (grid_used) *grid_used = g.grid;
    switch (f) {
      case 4: {
        const cudaError_t e = launch_pass_c4(c, p->LZ, p->LT, g.cp, mode, g.grid, g.smem, st);
        if (e != cudaErrorNotSupported) return e;
        cudaGetLastError();
        f = p->kc[2][mode].cp ? 3 : p->kc[1][mode].cp ? 2 : 1;
        continue;
      }
      case 3: return launch_pass_c3(c, p->LZ, p->LT, g.cp, g.grid, g.smem, st);
      case 2: return launch_pass_c2(c, p->LZ, p->LT, g.cp, mode, g.grid, g.smem, st);
      default: return launch_pass_c(c, p->LZ, p->LT, mode, g.grid, g.smem, st);
    }
  }
}

fno_status check_ready(fno_plan_t p, const char* who) {
  if (!p) return fail(FNO_ERR_INVALID_ARGUMENT, std::string(who) + ": NULL plan");
  if (!p->ws) return fail(FNO_ERR_INVALID_STATE, std::string(who) + ": workspace not set (fno_plan_set_workspace)");
  if (p->P > 1 && !p->group && (!p->comm || !p->comm->nccl))
    return fail(FNO_ERR_INVALID_STATE, std::string(who) + ": communicator missing");
  return FNO_OK;
}

#define FNO_TRY(x)                \
  do {                            \
    fno_status _s = (x);          \
    if (_s != FNO_OK) return _s;  \
  } while (0)

// ---- the layer as stages ----------------------------------------------------
// A stage is a sequence of this rank's launches that never waits for another
// rank; the exchanges sit between stages.  One process per GPU runs the stages
// of one plan back to back with the exchanges in between; a plan group
// (fno_group_*, one device) runs each stage for every rank before the next.

// forward, stage A: pass A (t, z transforms of v, I_1) -> the kz owners' slabs
fno_status sf_stage_a(fno_plan_t p, const float* v, cudaStream_t st) { return run_pass_a(p, v, nullptr, MODE_V, st); }

// forward, stage B: pass B on the owned kz block (y, x forward -> V^; mixing
// with R on the owned modes; x, y inverse -> the x/y owners' slabs)
fno_status sf_stage_b(fno_plan_t p, const float2* R, float2* vhat, cudaStream_t st) {
  FNO_TRY(run_b_fwd(p, vhat, st));
  if (p->nkz > 0) {
    MixParams m = make_mix(p);
    m.vhat = vhat; m.R = R; m.what = wsp<float2>(p, p->o_what);
    FNO_LAUNCH(p, ST_MIX, launch_mix_fwd(m, st), "mixing (forward)");
  }
  return run_b_inv(p, wsp<float2>(p, p->o_what), st);
}

// adjoint, stage A: pass A on g (or dz = dy sigma'(z) when mode says so)
fno_status sb_stage_a(fno_plan_t p, const float* in0, const float* in1, int mode, cudaStream_t st) {
  return run_pass_a(p, in0, in1, mode, st);
}

// adjoint, stage B: pass B with R^H, and dR on the owned modes (no comm)
fno_status sb_stage_b(fno_plan_t p, const float2* R, const float2* vhat_saved, float2* dR, int accumulate,
                      cudaStream_t st) {
  float2* ghat = wsp<float2>(p, p->o_ghat);
  FNO_TRY(run_b_fwd(p, ghat, st));
  if (p->nkz > 0) {
    MixParams m = make_mix(p);
    m.vhat = vhat_saved; m.R = R; m.ghat = ghat; m.what = wsp<float2>(p, p->o_what);
    m.dR = dR; m.accumulate = accumulate;
    FNO_LAUNCH(p, ST_MIX, launch_mix_bwd(m, st), "mixing (backward)");
  }
  return run_b_inv(p, wsp<float2>(p, p->o_what), st);
}

// stage C: pass C (inverse z, t) with the plain output u = S v (or S^T g)
fno_status stage_c_u(fno_plan_t p, float* out, cudaStream_t st) {
  PassCParams c = make_c(p, EPI_U);
  c.out = out;
  FNO_LAUNCH(p, ST_PASS_C, run_pass_c(p, c, EPI_U, st), "pass C (u)");
  return FNO_OK;
}

// stage C of the layer forward: z = W v + b + u, y = sigma(z)
fno_status stage_c_fwd(fno_plan_t p, const float* v, const float* W, const float* b, float* y, float* z_save,
                       cudaStream_t st) {
  PassCParams c = make_c(p, EPI_FWD);
  c.v = v; c.W = W; c.bias = b; c.out = y; c.zsave = z_save;
  FNO_LAUNCH(p, ST_PASS_C, run_pass_c(p, c, EPI_FWD, st), "pass C (layer forward)");
  return FNO_OK;
}

// stage C of the layer backward: dv = W^T dz + S^T dz and the per-CTA dW / db
// partials; then this rank's fixed-order partial sum (into `loc`, or straight
// into dW / db when loc is NULL)
fno_status stage_c_bwd(fno_plan_t p, const float* v, const float* dz, const float* W, float* dv, float* loc, float* dW,
                       float* db, int accumulate, cudaStream_t st) {
  int nparts = 1;
  if (p->fam[EPI_BWD] == 5) {
    // split backward: dv = W^T dz + S^T dz by the forward-mode kernel (the
    // contraction with W^T, no bias, identity, no z), then dW / db from dz, v
    PassCParams c = make_c(p, EPI_FWD);
    c.v = dz; c.W = W; c.w_t = 1; c.bias = nullptr; c.act_gelu = 0; c.zsave = nullptr; c.out = dv;
    FNO_LAUNCH(p, ST_PASS_C, run_pass_c(p, c, EPI_FWD, st), "pass C (layer backward, dv)");
    DwParams d{};
    d.dz = dz; d.v = v; d.part = wsp<float>(p, p->o_dwpart);
    d.N = p->Xl * p->Yl * p->Z * p->T; d.B = p->B; d.C = p->C;
    FNO_LAUNCH(p, ST_DWP, launch_dw_partial(d, p->dw_grid, st), "dW/db partials");
    nparts = p->dw_grid;
  } else {
    PassCParams c = make_c(p, EPI_BWD);
    c.v = v; c.dy = dz; c.W = W; c.out = dv;
    FNO_LAUNCH(p, ST_PASS_C, run_pass_c(p, c, EPI_BWD, st, &nparts), "pass C (layer backward)");
  }
  const float* dWpart = wsp<float>(p, p->o_dwpart);
  const int len = p->C * p->C + p->C;
  if (!loc) {
    FNO_LAUNCH(p, ST_DW, launch_rowsum(dWpart, nparts, len, p->C * p->C, dW, db, accumulate, st), "dW/db reduction");
  } else {
    FNO_LAUNCH(p, ST_DW, launch_rowsum(dWpart, nparts, len, len, loc, nullptr, 0, st), "dW/db local reduction");
  }
  return FNO_OK;
}

// forward spectral chain up to the second exchange; the slab for pass C is
// left in the x/y-ordered buffer.  vhat: where V^ goes (scratch or saved).
fno_status spectral_fwd_to_slab(fno_plan_t p, const float* v, const float2* R, float2* vhat, cudaStream_t st) {
  FNO_TRY(sf_stage_a(p, v, st));
  FNO_TRY(exchange_fwd(p, st));
  FNO_TRY(sf_stage_b(p, R, vhat, st));
  return exchange_bwd(p, st);
}

// adjoint spectral chain on g (input already in the pass-A form selected by mode)
fno_status spectral_bwd_to_slab(fno_plan_t p, const float* in0, const float* in1, int mode, const float2* R,
                                const float2* vhat_saved, float2* dR, int accumulate, cudaStream_t st) {
  FNO_TRY(sb_stage_a(p, in0, in1, mode, st));
  FNO_TRY(exchange_fwd(p, st));
  FNO_TRY(sb_stage_b(p, R, vhat_saved, dR, accumulate, st));
  return exchange_bwd(p, st);
}

fno_status not_grouped(fno_plan_t p, const char* who) {
  if (p && p->group) return fail(FNO_ERR_INVALID_STATE, std::string(who) + ": the plan belongs to a plan group (use fno_group_*)");
  return FNO_OK;
}

}  // namespace

static fno_status xy_spectral_conv_fwd(fno_plan_t p, const float* v, const void* R, float* u, void* vhat_save,
                                       void* stream) {
  FNO_TRY(check_ready(p, "fno_spectral_conv_fwd"));
  FNO_TRY(not_grouped(p, "fno_spectral_conv_fwd"));
  p->dir = 0;
  if (!v || !u || (!R && p->nkz > 0)) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_spectral_conv_fwd: NULL data pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float2* vhat = vhat_save ? static_cast<float2*>(vhat_save) : wsp<float2>(p, p->o_vhat);
  FNO_TRY(spectral_fwd_to_slab(p, v, static_cast<const float2*>(R), vhat, st));
  return stage_c_u(p, u, st);
}

static fno_status xy_spectral_conv_bwd(fno_plan_t p, const float* g, const void* R, const void* vhat_saved,
                                       float* dv, void* dR, int accumulate, void* stream) {
  FNO_TRY(check_ready(p, "fno_spectral_conv_bwd"));
  FNO_TRY(not_grouped(p, "fno_spectral_conv_bwd"));
  p->dir = 1;
  if (!g || (!R && p->nkz > 0)) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_spectral_conv_bwd: NULL g or R");
  if (dR && !vhat_saved && p->nkz > 0) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_spectral_conv_bwd: dR requires vhat_saved");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  FNO_TRY(spectral_bwd_to_slab(p, g, nullptr, MODE_V, static_cast<const float2*>(R), static_cast<const float2*>(vhat_saved),
                               static_cast<float2*>(dR), accumulate, st));
  if (dv) FNO_TRY(stage_c_u(p, dv, st));
  return FNO_OK;
}

static fno_status xy_layer_fwd(fno_plan_t p, const float* v, const void* R, const float* W, const float* b, float* y,
                               float* z_save, void* vhat_save, void* stream) {
  FNO_TRY(check_ready(p, "fno_layer_fwd"));
  FNO_TRY(not_grouped(p, "fno_layer_fwd"));
  p->dir = 0;
  if (!v || !W || !y || (!R && p->nkz > 0)) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_layer_fwd: NULL data pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float2* vhat = vhat_save ? static_cast<float2*>(vhat_save) : wsp<float2>(p, p->o_vhat);
  FNO_TRY(spectral_fwd_to_slab(p, v, static_cast<const float2*>(R), vhat, st));
  return stage_c_fwd(p, v, W, b, y, z_save, st);
}

static fno_status xy_layer_bwd(fno_plan_t p, const float* v, const float* z_saved, const void* vhat_saved,
                               const float* dy, const void* R, const float* W, float* dv, void* dR, float* dW,
                               float* db, int accumulate, void* stream) {
  FNO_TRY(check_ready(p, "fno_layer_bwd"));
  FNO_TRY(not_grouped(p, "fno_layer_bwd"));
  p->dir = 1;
  if (!v || !dy || !W || !dv || !dW || (!R && p->nkz > 0) || (p->act_gelu && !z_saved))
    return fail(FNO_ERR_INVALID_ARGUMENT, "fno_layer_bwd: NULL data pointer (v, dy, W, dv, dW, R and z_saved for GELU are required)");
  if (dR && !vhat_saved && p->nkz > 0) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_layer_bwd: dR requires vhat_saved");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int mode = p->act_gelu ? MODE_DZ_GELU : MODE_DZ_NONE;
  FNO_TRY(spectral_bwd_to_slab(p, dy, z_saved, mode, static_cast<const float2*>(R), static_cast<const float2*>(vhat_saved),
                               static_cast<float2*>(dR), accumulate, st));
  const float* dz = p->act_gelu ? wsp<float>(p, p->o_dz) : dy;   // dz formed by pass A
  if (p->P == 1) return stage_c_bwd(p, v, dz, W, dv, nullptr, dW, db, accumulate, st);
  float* loc = wsp<float>(p, p->o_dwloc);
  float* all = wsp<float>(p, p->o_dwall);
  FNO_TRY(stage_c_bwd(p, v, dz, W, dv, loc, nullptr, nullptr, 0, st));
  const int len = p->C * p->C + p->C;
  FNO_NCCL(ncclAllGather(loc, all, size_t(len), ncclFloat, p->comm->nccl, st), "dW/db all-gather");
  FNO_LAUNCH(p, ST_DW, launch_rowsum(all, p->P, len, p->C * p->C, dW, db, accumulate, st), "dW/db rank-ordered sum");
  return FNO_OK;
}

// ---------------------------------------------------------------------------
// plan groups: the P ranks of a decomposition as P plans in ONE process on ONE
// device (fno_group_*).  The data path is the decomposed one -- every rank's
// x/y box, the send-ready slab chunks stored straight into the owners' buffers
// (the peer-store exchange, with same-device pointers), kz-owned weights and
// the rank-ordered dW / db sum -- with each stage run for every rank before the
// next stage, so no rank ever waits for another (stream order is the barrier).
// ---------------------------------------------------------------------------
namespace {

bool same_problem(const fno_problem& a, const fno_problem& b) {
  for (int d = 0; d < 4; ++d)
    if (a.grid[d] != b.grid[d] || a.modes[d] != b.modes[d]) return false;
  return a.batch == b.batch && a.width == b.width && a.pgrid[0] == b.pgrid[0] && a.pgrid[1] == b.pgrid[1] &&
         a.flags == b.flags;
}

fno_status check_group(int n, fno_plan_t const* plans, const char* who) {
  if (n < 1 || !plans) return fail(FNO_ERR_INVALID_ARGUMENT, std::string(who) + ": need n >= 1 plans");
  for (int r = 0; r < n; ++r) {
    fno_plan_t p = plans[r];
    if (!p) return fail(FNO_ERR_INVALID_ARGUMENT, std::string(who) + ": NULL plan");
    if (!p->group || p->P != n || p->rank != r)
      return fail(FNO_ERR_INVALID_STATE, std::string(who) + ": plans must be a connected group in rank order (fno_group_connect)");
  }
  return FNO_OK;
}

}  // namespace

extern "C" fno_status fno_group_connect(int n, fno_plan_t* plans) {
  if (n < 1 || n > FNO_MAXP || !plans) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_group_connect: need 1 <= n <= 64 plans");
  int dev0 = -1;
  for (int r = 0; r < n; ++r) {
    fno_plan_t p = plans[r];
    if (!p) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_group_connect: NULL plan");
    if (p->P != n || p->rank != r) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_group_connect: plan r must be rank r of an n-rank problem");
    if (!same_problem(p->pb, plans[0]->pb)) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_group_connect: plans of different problems");
    if (!p->ws) return fail(FNO_ERR_INVALID_STATE, "fno_group_connect: workspace not set");
    if (p->peer || p->io_on) return fail(FNO_ERR_INVALID_STATE, "fno_group_connect: plan already connected or io-partitioned");
    cudaPointerAttributes at{};
    FNO_CUDA(cudaPointerGetAttributes(&at, p->ws), "fno_group_connect: workspace attributes");
    if (at.type != cudaMemoryTypeDevice) return fail(FNO_ERR_WORKSPACE, "fno_group_connect: workspace is not device memory");
    if (dev0 < 0) dev0 = at.device;
    if (at.device != dev0) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_group_connect: all workspaces must be on one device");
  }
  std::vector<char*> bases(n);
  for (int r = 0; r < n; ++r) bases[r] = static_cast<char*>(plans[r]->ws);
  for (int r = 0; r < n; ++r) {
    plans[r]->peer_ws = bases;
    plans[r]->peer = n > 1 ? 1 : 0;
    plans[r]->group = 1;
  }
  return FNO_OK;
}

extern "C" fno_status fno_group_spectral_conv_fwd(int n, fno_plan_t* plans, const float* const* v, const void* const* R,
                                                  float* const* u, void* const* vhat_save, void* stream) {
  FNO_TRY(check_group(n, plans, "fno_group_spectral_conv_fwd"));
  if (!v || !R || !u) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_group_spectral_conv_fwd: NULL array");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  auto vh = [&](int r) { return vhat_save && vhat_save[r] ? static_cast<float2*>(vhat_save[r]) : wsp<float2>(plans[r], plans[r]->o_vhat); };
  for (int r = 0; r < n; ++r) { plans[r]->dir = 0; FNO_TRY(sf_stage_a(plans[r], v[r], st)); }
  for (int r = 0; r < n; ++r) FNO_TRY(sf_stage_b(plans[r], static_cast<const float2*>(R[r]), vh(r), st));
  for (int r = 0; r < n; ++r) FNO_TRY(stage_c_u(plans[r], u[r], st));
  return FNO_OK;
}

extern "C" fno_status fno_group_spectral_conv_bwd(int n, fno_plan_t* plans, const float* const* g, const void* const* R,
                                                  const void* const* vhat_saved, float* const* dv, void* const* dR,
                                                  int accumulate, void* stream) {
  FNO_TRY(check_group(n, plans, "fno_group_spectral_conv_bwd"));
  if (!g || !R) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_group_spectral_conv_bwd: NULL array");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (int r = 0; r < n; ++r) { plans[r]->dir = 1; FNO_TRY(sb_stage_a(plans[r], g[r], nullptr, MODE_V, st)); }
  for (int r = 0; r < n; ++r)
    FNO_TRY(sb_stage_b(plans[r], static_cast<const float2*>(R[r]), vhat_saved ? static_cast<const float2*>(vhat_saved[r]) : nullptr,
                       dR ? static_cast<float2*>(dR[r]) : nullptr, accumulate, st));
  if (dv)
    for (int r = 0; r < n; ++r) FNO_TRY(stage_c_u(plans[r], dv[r], st));
  return FNO_OK;
}

extern "C" fno_status fno_group_layer_fwd(int n, fno_plan_t* plans, const float* const* v, const void* const* R,
                                          const float* W, const float* b, float* const* y, float* const* z_save,
                                          void* const* vhat_save, void* stream) {
  FNO_TRY(check_group(n, plans, "fno_group_layer_fwd"));
  if (!v || !R || !W || !y) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_group_layer_fwd: NULL argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  auto vh = [&](int r) { return vhat_save && vhat_save[r] ? static_cast<float2*>(vhat_save[r]) : wsp<float2>(plans[r], plans[r]->o_vhat); };
  for (int r = 0; r < n; ++r) { plans[r]->dir = 0; FNO_TRY(sf_stage_a(plans[r], v[r], st)); }
  for (int r = 0; r < n; ++r) FNO_TRY(sf_stage_b(plans[r], static_cast<const float2*>(R[r]), vh(r), st));
  for (int r = 0; r < n; ++r) FNO_TRY(stage_c_fwd(plans[r], v[r], W, b, y[r], z_save ? z_save[r] : nullptr, st));
  return FNO_OK;
}

extern "C" fno_status fno_group_layer_bwd(int n, fno_plan_t* plans, const float* const* v, const float* const* z_saved,
                                          const void* const* vhat_saved, const float* const* dy, const void* const* R,
                                          const float* W, float* const* dv, void* const* dR, float* dW, float* db,
                                          int accumulate, void* stream) {
  FNO_TRY(check_group(n, plans, "fno_group_layer_bwd"));
  const int act = plans[0]->act_gelu;
  if (!v || !dy || !R || !W || !dv || !dW || !vhat_saved || (act && !z_saved))
    return fail(FNO_ERR_INVALID_ARGUMENT, "fno_group_layer_bwd: NULL argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int mode = act ? MODE_DZ_GELU : MODE_DZ_NONE;
  for (int r = 0; r < n; ++r) { plans[r]->dir = 1; FNO_TRY(sb_stage_a(plans[r], dy[r], act ? z_saved[r] : nullptr, mode, st)); }
  for (int r = 0; r < n; ++r)
    FNO_TRY(sb_stage_b(plans[r], static_cast<const float2*>(R[r]), static_cast<const float2*>(vhat_saved[r]),
                       dR ? static_cast<float2*>(dR[r]) : nullptr, accumulate, st));
  const int len = plans[0]->C * plans[0]->C + plans[0]->C;
  float* all = wsp<float>(plans[0], plans[0]->o_dwall);
  for (int r = 0; r < n; ++r) {
    fno_plan_t p = plans[r];
    const float* dz = act ? wsp<float>(p, p->o_dz) : dy[r];
    float* loc = wsp<float>(p, p->o_dwloc);
    FNO_TRY(stage_c_bwd(p, v[r], dz, W, dv[r], loc, nullptr, nullptr, 0, st));
    FNO_CUDA(cudaMemcpyAsync(all + size_t(r) * len, loc, size_t(len) * sizeof(float), cudaMemcpyDeviceToDevice, st),
             "group: dW/db gather");
  }
  FNO_LAUNCH(plans[0], ST_DW, launch_rowsum(all, n, len, plans[0]->C * plans[0]->C, dW, db, accumulate, st),
             "group: dW/db rank-ordered sum");
  return FNO_OK;
}

// ---------------------------------------------------------------------------
// caller-side partitions other than the plan's x/y grid (App. A
// 3-D spatial and temporal partitions): every field is repartitioned
// to the x/y grid on entry and back on exit ("a repartition operator is
// used to take the data to a partition of only the x and y dimensions")
// ---------------------------------------------------------------------------
fno_status io_move(fno_plan_t p, const float* src, float* dst, bool to_xy, cudaStream_t st) {
  const int64_t shape[6] = {p->B, p->C, p->X, p->Y, p->Z, p->T};
  const int32_t io6[6] = {1, 1, p->io[0], p->io[1], p->io[2], p->io[3]};
  const int32_t xy6[6] = {1, 1, p->px, p->py, 1, 1};
  size_t wsb = p->io_ws_bytes;
  return fno_repartition(p->comm, 6, shape, to_xy ? io6 : xy6, to_xy ? xy6 : io6, sizeof(float), src, dst,
                         wsp<void>(p, p->o_io_ws), &wsb, st);
}

extern "C" fno_status fno_plan_set_io_partition(fno_plan_t p, const int32_t io_pgrid[4]) {
  if (!p || !io_pgrid) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_plan_set_io_partition: NULL argument");
  if (p->ws) return fail(FNO_ERR_INVALID_STATE, "fno_plan_set_io_partition: call before fno_plan_set_workspace");
  if (p->io_on) return fail(FNO_ERR_INVALID_STATE, "fno_plan_set_io_partition: already set");
  if (p->peer) return fail(FNO_ERR_INVALID_STATE, "fno_plan_set_io_partition: call before fno_plan_connect_peers");
  const long long ext[4] = {p->X, p->Y, p->Z, p->T};
  long long prod = 1;
  for (int d = 0; d < 4; ++d) {
    if (io_pgrid[d] < 1 || ext[d] % io_pgrid[d] != 0)
      return fail(FNO_ERR_INVALID_ARGUMENT, "fno_plan_set_io_partition: every extent must be divisible by its partition");
    prod *= io_pgrid[d];
  }
  if (prod != p->P) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_plan_set_io_partition: partition size must equal the plan's ranks");
  for (int d = 0; d < 4; ++d) p->io[d] = io_pgrid[d];
  if (io_pgrid[0] == p->px && io_pgrid[1] == p->py && io_pgrid[2] == 1 && io_pgrid[3] == 1) return FNO_OK;
  p->io_on = true;
  const int64_t shape[6] = {p->B, p->C, p->X, p->Y, p->Z, p->T};
  const int32_t io6[6] = {1, 1, p->io[0], p->io[1], p->io[2], p->io[3]};
  const int32_t xy6[6] = {1, 1, p->px, p->py, 1, 1};
  size_t a = 0, b = 0;
  FNO_TRY(fno_repartition(p->comm, 6, shape, io6, xy6, sizeof(float), nullptr, nullptr, nullptr, &a, nullptr));
  FNO_TRY(fno_repartition(p->comm, 6, shape, xy6, io6, sizeof(float), nullptr, nullptr, nullptr, &b, nullptr));
  const size_t field = align256(size_t(p->B) * p->C * p->Xl * p->Yl * p->Z * p->T * sizeof(float));
  p->io_ws_bytes = std::max(a, b);
  p->o_io_a = p->total;
  p->o_io_b = p->o_io_a + field;
  p->o_io_c = p->o_io_b + field;
  p->o_io_ws = p->o_io_c + field;
  p->total = p->o_io_ws + align256(p->io_ws_bytes);
  return FNO_OK;
}

extern "C" fno_status fno_plan_io_box(fno_plan_t p, int64_t lo[4], int64_t hi[4]) {
  if (!p || !lo || !hi) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_plan_io_box: NULL argument");
  const long long ext[4] = {p->X, p->Y, p->Z, p->T};
  int r = p->rank;
  int coords[4];
  for (int d = 3; d >= 0; --d) {
    coords[d] = r % p->io[d];
    r /= p->io[d];
  }
  for (int d = 0; d < 4; ++d) {
    long long l, h;
    block_range(ext[d], p->io[d], coords[d], &l, &h);
    lo[d] = l;
    hi[d] = h;
  }
  return FNO_OK;
}

extern "C" fno_status fno_spectral_conv_fwd(fno_plan_t p, const float* v, const void* R, float* u, void* vhat_save,
                                            void* stream) {
  if (!p || !p->io_on) return xy_spectral_conv_fwd(p, v, R, u, vhat_save, stream);
  FNO_TRY(check_ready(p, "fno_spectral_conv_fwd"));
  if (!v || !u) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_spectral_conv_fwd: NULL data pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float* va = wsp<float>(p, p->o_io_a);
  float* ub = wsp<float>(p, p->o_io_b);
  FNO_TRY(io_move(p, v, va, true, st));
  FNO_TRY(xy_spectral_conv_fwd(p, va, R, ub, vhat_save, stream));
  return io_move(p, ub, u, false, st);
}

extern "C" fno_status fno_spectral_conv_bwd(fno_plan_t p, const float* g, const void* R, const void* vhat_saved,
                                            float* dv, void* dR, int accumulate, void* stream) {
  if (!p || !p->io_on) return xy_spectral_conv_bwd(p, g, R, vhat_saved, dv, dR, accumulate, stream);
  FNO_TRY(check_ready(p, "fno_spectral_conv_bwd"));
  if (!g) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_spectral_conv_bwd: NULL g");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float* ga = wsp<float>(p, p->o_io_a);
  float* db = wsp<float>(p, p->o_io_b);
  FNO_TRY(io_move(p, g, ga, true, st));
  FNO_TRY(xy_spectral_conv_bwd(p, ga, R, vhat_saved, dv ? db : nullptr, dR, accumulate, stream));
  if (dv) FNO_TRY(io_move(p, db, dv, false, st));
  return FNO_OK;
}

// z_save / z_saved stay in the plan's x/y layout (an opaque buffer of the same size)
extern "C" fno_status fno_layer_fwd(fno_plan_t p, const float* v, const void* R, const float* W, const float* b, float* y,
                                    float* z_save, void* vhat_save, void* stream) {
  if (!p || !p->io_on) return xy_layer_fwd(p, v, R, W, b, y, z_save, vhat_save, stream);
  FNO_TRY(check_ready(p, "fno_layer_fwd"));
  if (!v || !y) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_layer_fwd: NULL data pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float* va = wsp<float>(p, p->o_io_a);
  float* yb = wsp<float>(p, p->o_io_b);
  FNO_TRY(io_move(p, v, va, true, st));
  FNO_TRY(xy_layer_fwd(p, va, R, W, b, yb, z_save, vhat_save, stream));
  return io_move(p, yb, y, false, st);
}

extern "C" fno_status fno_layer_bwd(fno_plan_t p, const float* v, const float* z_saved, const void* vhat_saved,
                                    const float* dy, const void* R, const float* W, float* dv, void* dR, float* dW,
                                    float* db, int accumulate, void* stream) {
  if (!p || !p->io_on) return xy_layer_bwd(p, v, z_saved, vhat_saved, dy, R, W, dv, dR, dW, db, accumulate, stream);
  FNO_TRY(check_ready(p, "fno_layer_bwd"));
  if (!v || !dy || !dv) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_layer_bwd: NULL data pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float* va = wsp<float>(p, p->o_io_a);
  float* dyb = wsp<float>(p, p->o_io_b);
  float* dvc = wsp<float>(p, p->o_io_c);
  FNO_TRY(io_move(p, v, va, true, st));
  FNO_TRY(io_move(p, dy, dyb, true, st));
  FNO_TRY(xy_layer_bwd(p, va, z_saved, vhat_saved, dyb, R, W, dvc, dR, dW, db, accumulate, stream));
  return io_move(p, dvc, dv, false, st);
}

// ---------------------------------------------------------------------------
// whole network
// ---------------------------------------------------------------------------
namespace {

// net workspace layout (bytes offsets), sized for the plan's local box
struct NetWs {
  size_t dloss, sums, dall, lparts, pparts, row, rall, total;
  int gl, gp, gb, plen;
};

NetWs net_ws_layout(fno_plan_t p, int Cin) {
  NetParams q{};
  q.B = p->B; q.C = p->C; q.Cin = Cin; q.T = int(p->T); q.NS = p->Xl * p->Yl * p->Z;
  NetWs w{};
  w.gl = net_loss_grid(q, p->num_sms);
  w.gp = net_proj_bwd_grid(q, p->num_sms);
  w.gb = net_lift_bwd_grid(q, p->num_sms);
  w.plen = p->C * Cin + p->C + 2 * int(p->T);
  const int rlen = std::max(w.plen, p->C + 1);
  size_t off = 0;
  auto take = [&](size_t b) { size_t o = off; off += align256(b); return o; };
  w.dloss = take(size_t(w.gl) * 2 * sizeof(double));
  w.sums = take(4 * sizeof(double));
  w.dall = take(size_t(p->P) * 2 * sizeof(double));
  w.lparts = take(size_t(w.gb) * w.plen * sizeof(float));
  w.pparts = take(size_t(w.gp) * (p->C + 1) * sizeof(float));
  w.row = take(size_t(rlen) * sizeof(float));
  w.rall = take(size_t(p->P) * rlen * sizeof(float));
  w.total = off;
  return w;
}

fno_status net_check(fno_plan_t p, const fno_net_desc* d, const char* who) {
  FNO_TRY(check_ready(p, who));
  if (!d || d->layers < 1 || d->layers > FNO_NET_MAXK || d->in_channels < 1 || d->in_channels > 4)
    return fail(FNO_ERR_INVALID_ARGUMENT, std::string(who) + ": need 1 <= layers <= FNO_NET_MAXK and 1 <= in_channels <= 4");
  if (p->C > 32) return fail(FNO_ERR_PLAN, std::string(who) + ": the network kernels support width C <= 32");
  if (p->io_on) return fail(FNO_ERR_INVALID_STATE, std::string(who) + ": the network runs on the plan's x/y partition (no io partition)");
  if ((p->Xl * p->Yl * p->Z * p->T) % 4 != 0)
    return fail(FNO_ERR_PLAN, std::string(who) + ": the network kernels need Xl*Yl*Z*T to be a multiple of 4");
  return FNO_OK;
}

NetParams net_base(fno_plan_t p, int Cin) {
  NetParams q{};
  q.B = p->B; q.C = p->C; q.Cin = Cin; q.T = int(p->T); q.NS = p->Xl * p->Yl * p->Z;
  return q;
}

// the replicated-parameter gradient row `row` (len floats, this rank's sum)
// summed over ranks in rank order into `out` (len floats); P == 1: copy
fno_status net_rank_sum(fno_plan_t p, float* row, int len, float* rall, float* out, cudaStream_t st) {
  if (p->P == 1) {
    FNO_CUDA(cudaMemcpyAsync(out, row, size_t(len) * sizeof(float), cudaMemcpyDeviceToDevice, st), "net: gradient copy");
    return FNO_OK;
  }
  FNO_NCCL(ncclAllGather(row, rall, size_t(len), ncclFloat, p->comm->nccl, st), "net: gradient all-gather");
  FNO_CUDA(launch_rowsum_strided(rall, p->P, len, len, out, 0, st), "net: rank-ordered gradient sum");
  g_launches++;
  return FNO_OK;
}

// runs one block with the activation of its position (GELU except the last)
struct ActScope {
  fno_plan_t p;
  int saved;
  ActScope(fno_plan_t p_, int act) : p(p_), saved(p_->act_gelu) { p->act_gelu = act; }
  ~ActScope() { p->act_gelu = saved; }
};

}  // namespace

extern "C" fno_status fno_net_workspace_size(fno_plan_t p, const fno_net_desc* d, size_t* bytes) {
  if (!p || !d || !bytes) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_net_workspace_size: NULL argument");
  if (d->in_channels < 1 || d->in_channels > 4) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_net_workspace_size: 1 <= in_channels <= 4");
  *bytes = net_ws_layout(p, d->in_channels).total;
  return FNO_OK;
}

extern "C" fno_status fno_net_fwd(fno_plan_t p, const fno_net_desc* d, const fno_net_params* w, const float* a,
                                  const fno_net_acts* acts, float* u, void* stream) {
  FNO_TRY(net_check(p, d, "fno_net_fwd"));
  if (!w || !a || !acts || !u || !w->Wt || !w->bt || !w->Wc || !w->bc || !w->Wp || (d->proj_bias && !w->bp))
    return fail(FNO_ERR_INVALID_ARGUMENT, "fno_net_fwd: NULL argument");
  const int K = d->layers;
  for (int k = 0; k <= K; ++k)
    if (!acts->nu[k]) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_net_fwd: acts->nu[k] is NULL");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  NetParams q = net_base(p, d->in_channels);
  q.a = a; q.Wt = w->Wt; q.bt = w->bt; q.Wc = w->Wc; q.bc = w->bc; q.nu = acts->nu[0];
  FNO_CUDA(launch_net_lift_fwd(q, p->num_sms, st), "net: lift");
  g_launches++;
  for (int k = 0; k < K; ++k) {
    const int act = k < K - 1 ? 1 : 0;
    if (act && !acts->z[k]) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_net_fwd: acts->z[k] is NULL for a GELU block");
    ActScope as(p, act);
    FNO_TRY(xy_layer_fwd(p, acts->nu[k], w->R[k], w->W[k], w->b[k], acts->nu[k + 1], act ? acts->z[k] : nullptr,
                          acts->vhat[k], stream));
  }
  q.nu = acts->nu[K]; q.Wp = w->Wp; q.bp = d->proj_bias ? w->bp : nullptr; q.u = u;
  FNO_CUDA(launch_net_proj_fwd(q, p->num_sms, st), "net: projection");
  g_launches++;
  return FNO_OK;
}

extern "C" fno_status fno_net_loss(fno_plan_t p, const float* u, const float* y, float* loss3, void* net_ws, void* stream) {
  FNO_TRY(check_ready(p, "fno_net_loss"));
  if (!u || !y || !loss3 || !net_ws) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_net_loss: NULL argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const NetWs L = net_ws_layout(p, 1);
  char* ws = static_cast<char*>(net_ws);
  NetParams q = net_base(p, 1);
  q.u = const_cast<float*>(u); q.y = y; q.dparts = reinterpret_cast<double*>(ws + L.dloss);
  double* sums = reinterpret_cast<double*>(ws + L.sums);
  FNO_CUDA(launch_net_loss_partial(q, L.gl, st), "net: loss partial sums");
  g_launches++;
  if (p->P == 1) {
    FNO_CUDA(launch_net_loss_finalize(q.dparts, L.gl, sums, loss3, st), "net: loss");
    g_launches++;
  } else {
    double* dall = reinterpret_cast<double*>(ws + L.dall);
    FNO_CUDA(launch_net_loss_finalize(q.dparts, L.gl, dall + 2 * p->rank, nullptr, st), "net: local loss sums");
    g_launches++;
    FNO_NCCL(ncclAllGather(dall + 2 * p->rank, dall, 2, ncclDouble, p->comm->nccl, st), "net: loss all-gather");
    FNO_CUDA(launch_net_loss_finalize(dall, p->P, sums, loss3, st), "net: loss (rank order)");
    g_launches++;
  }
  return FNO_OK;
}

extern "C" fno_status fno_net_bwd(fno_plan_t p, const fno_net_desc* d, const fno_net_params* w, const float* a,
                                  const fno_net_acts* acts, const float* u, const float* y, const fno_net_params* g,
                                  float* s0, float* s1, void* net_ws, void* stream) {
  FNO_TRY(net_check(p, d, "fno_net_bwd"));
  if (!w || !a || !acts || !u || !y || !g || !s0 || !s1 || !net_ws || !g->Wt || !g->bt || !g->Wc || !g->bc || !g->Wp ||
      (d->proj_bias && !g->bp))
    return fail(FNO_ERR_INVALID_ARGUMENT, "fno_net_bwd: NULL argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int K = d->layers, Cin = d->in_channels, C = p->C, T = int(p->T);
  // the fp64 loss sums of fno_net_loss sit at the same offset for every C_in
  const NetWs L = net_ws_layout(p, Cin);
  char* ws = static_cast<char*>(net_ws);
  float* row = reinterpret_cast<float*>(ws + L.row);
  float* rall = reinterpret_cast<float*>(ws + L.rall);
  NetParams q = net_base(p, Cin);
  // projection + loss adjoint -> dnu_K (s0), dWp, dbp
  q.u = const_cast<float*>(u); q.y = y; q.nu = acts->nu[K]; q.Wp = w->Wp; q.dnu = s0;
  q.parts = reinterpret_cast<float*>(ws + L.pparts); q.stats = reinterpret_cast<const double*>(ws + L.sums);
  FNO_CUDA(launch_net_proj_bwd(q, L.gp, st), "net: projection / loss adjoint");
  g_launches++;
  FNO_CUDA(launch_rowsum_strided(q.parts, L.gp, C + 1, C + 1, row, 0, st), "net: dWp / dbp partial sum");
  g_launches++;
  FNO_TRY(net_rank_sum(p, row, C, rall, g->Wp, st));
  if (d->proj_bias) FNO_TRY(net_rank_sum(p, row + C, 1, rall, g->bp, st));
  // blocks, last to first (ping-pong s0 -> s1 -> s0 ...)
  float* dcur = s0;
  float* dnext = s1;
  for (int k = K - 1; k >= 0; --k) {
    const int act = k < K - 1 ? 1 : 0;
    ActScope as(p, act);
    FNO_TRY(xy_layer_bwd(p, acts->nu[k], act ? acts->z[k] : nullptr, acts->vhat[k], dcur, w->R[k], w->W[k], dnext,
                          g->R[k], g->W[k], g->b[k], 0, stream));
    std::swap(dcur, dnext);
  }
  // lift adjoint -> dWc, dbc, dWt, dbt
  q.a = a; q.Wt = w->Wt; q.bt = w->bt; q.Wc = w->Wc; q.dnu = dcur;
  q.parts = reinterpret_cast<float*>(ws + L.lparts); q.plen = L.plen;
  FNO_CUDA(launch_net_lift_bwd(q, L.gb, st), "net: lift adjoint");
  g_launches++;
  FNO_CUDA(launch_rowsum_strided(q.parts, L.gb, L.plen, L.plen, row, 0, st), "net: lift gradient partial sum");
  g_launches++;
  FNO_TRY(net_rank_sum(p, row, C * Cin, rall, g->Wc, st));
  FNO_TRY(net_rank_sum(p, row + C * Cin, C, rall + size_t(p->P) * C * Cin, g->bc, st));
  FNO_TRY(net_rank_sum(p, row + C * Cin + C, T, rall + size_t(p->P) * (C * Cin + C), g->Wt, st));
  FNO_TRY(net_rank_sum(p, row + C * Cin + C + T, T, rall + size_t(p->P) * (C * Cin + C + T), g->bt, st));
  return FNO_OK;
}

extern "C" fno_status fno_comm_allreduce(fno_comm_t comm, float* buf, size_t n, int average, void* stream) {
  if (!comm || !comm->nccl) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_comm_allreduce: NULL communicator");
  if (n == 0) return FNO_OK;
  if (!buf) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_comm_allreduce: NULL buffer");
  FNO_NCCL(ncclAllReduce(buf, buf, n, ncclFloat, average ? ncclAvg : ncclSum, comm->nccl,
                         static_cast<cudaStream_t>(stream)), "fno_comm_allreduce");
  return FNO_OK;
}

extern "C" fno_status fno_adam(float* prm, const float* grad, float* m, float* v, size_t n, float lr, float beta1,
                               float beta2, float eps, int step, void* stream) {
  if (n == 0) return FNO_OK;
  if (!prm || !grad || !m || !v || step < 1) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_adam: NULL pointer or step < 1");
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  FNO_CUDA(launch_adam(prm, grad, m, v, (long long)n, lr, beta1, beta2, eps, step, sms, static_cast<cudaStream_t>(stream)),
           "adam");
  g_launches++;
  return FNO_OK;
}

// ---------------------------------------------------------------------------
// general repartition R_{P->Q}
// ---------------------------------------------------------------------------
namespace {

struct Box {
  long long lo[8], hi[8];
};

Box box_of(int ndim, const int64_t* shape, const int32_t* pg, int rank) {
  Box b{};
  int coords[8];
  int r = rank;
  for (int d = ndim - 1; d >= 0; --d) {
    coords[d] = r % pg[d];
    r /= pg[d];
  }
  for (int d = 0; d < ndim; ++d) block_range(shape[d], pg[d], coords[d], &b.lo[d], &b.hi[d]);
  return b;
}

bool intersect(int ndim, const Box& a, const Box& b, Box* o) {
  for (int d = 0; d < ndim; ++d) {
    o->lo[d] = std::max(a.lo[d], b.lo[d]);
    o->hi[d] = std::min(a.hi[d], b.hi[d]);
    if (o->lo[d] >= o->hi[d]) return false;
  }
  return true;
}

long long box_elems(int ndim, const Box& b) {
  long long n = 1;
  for (int d = 0; d < ndim; ++d) n *= (b.hi[d] - b.lo[d]);
  return n;
}

}  // namespace

cudaError_t launch_box_copy(const void* src, const long long* src_ext, const long long* src_lo, void* dst,
                            const long long* dst_ext, const long long* dst_lo, const long long* cnt, int ndim,
                            size_t elem_bytes, cudaStream_t st);

extern "C" fno_status fno_repartition(fno_comm_t comm, int ndim, const int64_t* shape, const int32_t* src_pg,
                                      const int32_t* dst_pg, size_t elem_bytes, const void* src_local, void* dst_local,
                                      void* workspace, size_t* ws_bytes, void* stream) {
  if (ndim < 1 || ndim > 8 || !shape || !src_pg || !dst_pg || !ws_bytes || elem_bytes == 0)
    return fail(FNO_ERR_INVALID_ARGUMENT, "fno_repartition: bad arguments (1 <= ndim <= 8, non-NULL shape/pgrids/ws_bytes)");
  int nranks = 1, rank = 0;
  if (comm) { nranks = comm->nranks; rank = comm->rank; }
  long long ns = 1, nd = 1;
  for (int d = 0; d < ndim; ++d) {
    if (shape[d] < 0 || src_pg[d] < 1 || dst_pg[d] < 1) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_repartition: bad shape or pgrid entry");
    ns *= src_pg[d];
    nd *= dst_pg[d];
  }
  if (ns != nranks || nd != nranks)
    return fail(FNO_ERR_INVALID_ARGUMENT, "fno_repartition: both partitions must have exactly comm-size workers");
  const Box mine_s = box_of(ndim, shape, src_pg, rank);
  const Box mine_d = box_of(ndim, shape, dst_pg, rank);
  // workspace: packed send [sum over peers] + packed recv [sum over peers]
  std::vector<long long> scount(nranks), rcount(nranks);
  std::vector<Box> sbox(nranks), rbox(nranks);
  long long stot = 0, rtot = 0;
  for (int q = 0; q < nranks; ++q) {
    Box o;
    scount[q] = intersect(ndim, mine_s, box_of(ndim, shape, dst_pg, q), &o) ? box_elems(ndim, o) : 0;
    sbox[q] = o;
    rcount[q] = intersect(ndim, box_of(ndim, shape, src_pg, q), mine_d, &o) ? box_elems(ndim, o) : 0;
    rbox[q] = o;
    stot += scount[q];
    rtot += rcount[q];
  }
  const size_t need = align256(size_t(stot) * elem_bytes) + align256(size_t(rtot) * elem_bytes);
  if (!workspace) {
    *ws_bytes = need;
    return FNO_OK;
  }
  if (*ws_bytes < need) return fail(FNO_ERR_WORKSPACE, "fno_repartition: workspace too small");
  if ((stot && !src_local) || (rtot && !dst_local)) return fail(FNO_ERR_INVALID_ARGUMENT, "fno_repartition: NULL local buffer");
  if (nranks > 1 && (!comm || !comm->nccl)) return fail(FNO_ERR_INVALID_STATE, "fno_repartition: communicator missing");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* sbuf = static_cast<char*>(workspace);
  char* rbuf = sbuf + align256(size_t(stot) * elem_bytes);
  long long sext[8], dext[8];
  for (int d = 0; d < ndim; ++d) {
    sext[d] = mine_s.hi[d] - mine_s.lo[d];
    dext[d] = mine_d.hi[d] - mine_d.lo[d];
  }
  // pack (peer order ascending)
  long long so = 0;
  for (int q = 0; q < nranks; ++q) {
    if (!scount[q]) continue;
    long long lo[8], cnt[8], zero[8] = {0};
    for (int d = 0; d < ndim; ++d) {
      lo[d] = sbox[q].lo[d] - mine_s.lo[d];
      cnt[d] = sbox[q].hi[d] - sbox[q].lo[d];
    }
    FNO_CUDA(launch_box_copy(src_local, sext, lo, sbuf + so * elem_bytes, cnt, zero, cnt, ndim, elem_bytes, st), "repartition pack");
    g_launches++;
    so += scount[q];
  }
  if (nranks > 1) {
    FNO_NCCL(ncclGroupStart(), "repartition: ncclGroupStart");
    long long s2 = 0, r2 = 0;
    for (int q = 0; q < nranks; ++q) {
      if (scount[q]) FNO_NCCL(ncclSend(sbuf + s2 * elem_bytes, size_t(scount[q]) * elem_bytes, ncclUint8, q, comm->nccl, st), "repartition: ncclSend");
      if (rcount[q]) FNO_NCCL(ncclRecv(rbuf + r2 * elem_bytes, size_t(rcount[q]) * elem_bytes, ncclUint8, q, comm->nccl, st), "repartition: ncclRecv");
      s2 += scount[q];
      r2 += rcount[q];
    }
    FNO_NCCL(ncclGroupEnd(), "repartition: ncclGroupEnd");
  } else if (stot) {
    FNO_CUDA(cudaMemcpyAsync(rbuf, sbuf, size_t(stot) * elem_bytes, cudaMemcpyDeviceToDevice, st), "repartition self copy");
  }
  // unpack
  long long ro = 0;
  for (int q = 0; q < nranks; ++q) {
    if (!rcount[q]) continue;
    long long lo[8], cnt[8], zero[8] = {0};
    for (int d = 0; d < ndim; ++d) {
      lo[d] = rbox[q].lo[d] - mine_d.lo[d];
      cnt[d] = rbox[q].hi[d] - rbox[q].lo[d];
    }
    FNO_CUDA(launch_box_copy(rbuf + ro * elem_bytes, cnt, zero, dst_local, dext, lo, cnt, ndim, elem_bytes, st), "repartition unpack");
    g_launches++;
    ro += rcount[q];
  }
  return FNO_OK;
}
