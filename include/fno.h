/*
 * libfno — C ABI of the B200-native hot path of the model-parallel FNO of
 * arXiv 2204.01205 (Grady et al.): the 4D (x, y, z, t) spectral-convolution
 * layer, forward and adjoint, domain-decomposed over x/y.
 *
 * Citations are PAPER.md lines ("P:<line>") of /root/reference/PAPER.md.
 *
 *   S v   = F^-1 (R_phi . F v)                              P:48-52 (Eq. 3)
 *   S_dist= F_dist^T (R_phi . F_dist v)
 *   block : y = sigma(W v + b + S v)                        P:159-169 (Eq. dist_block)
 *   R_{P->Q} repartition (generalised all-to-all),
 *            adjoint R_{Q->P}
 *
 * Conventions:
 *   - Fields are NCXYZT, t fastest: float [B][C][Xl][Yl][Z][T], the
 *     caller's local x/y box (fno_plan_local_box).
 *   - Retained modes per spatial axis: {0..m-1} ∪ {n-m..n-1} (reading
 *     Q2), retained index j -> k = j (j < m) else n - 2m + j.  Along t the
 *     transform is real (rFFT) and keeps {0..mt-1} (readings Q1, Q2).
 *   - Forward transform unnormalised, inverse scaled by 1/(X Y Z T) (Q3);
 *     the inverse along t takes the real part with weights c(kt) = 1 at kt=0
 *     and at the Nyquist kt=T/2, 2 otherwise (real-part semantics, Q4).
 *   - Spectral weights R (and dR): complex64 (float2 {re, im})
 *     [C_in][C_out][2mx][2my][kz_hi-kz_lo][mt], the rank's block of retained
 *     kz planes (fno_plan_owned_modes).  Mixing: W^[o,k] = sum_i V^[i,k] R[i,o,k].
 *   - Channel weight W: float [C_out][C_in], replicated on every rank
 *     (broadcast weights); b: float [C] or NULL (= 0).
 *   - Process grid (1,1,px,py,1,1): rank = ix*py + iy (row-major, Q11).
 *
 * Ownership: the library NEVER allocates device memory.  Every data pointer is
 * device memory on the plan's device, owned by the caller.  The caller also
 * provides the workspace (fno_plan_workspace_size / fno_plan_set_workspace).
 * Plans own host metadata and a reference to the communicator only.
 *
 * Ordering: every compute call is asynchronous and stream-ordered on `stream`
 * (a cudaStream_t passed as void*; NULL = legacy default stream).  With P > 1,
 * every call is collective: all ranks must issue the same sequence of calls.
 *
 * Errors: every entry point returns fno_status; it never throws across the
 * ABI.  Argument errors are detected before any work is enqueued.  CUDA and
 * NCCL launch errors are returned as FNO_ERR_CUDA / FNO_ERR_NCCL; asynchronous
 * device faults surface on a later call or at the caller's synchronisation.
 * fno_last_error() returns a thread-local message naming the failing stage.
 */
#ifndef FNO_H_
#define FNO_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FNO_ABI_VERSION 1

typedef enum {
  FNO_OK = 0,
  FNO_ERR_INVALID_ARGUMENT = 1, /* bad shape, modes, pointer, partition      */
  FNO_ERR_PLAN = 2,             /* unplaceable partition / unsupported shape */
  FNO_ERR_INVALID_STATE = 3,    /* e.g. workspace not set, comm missing      */
  FNO_ERR_CUDA = 4,             /* a CUDA runtime call or launch failed      */
  FNO_ERR_NCCL = 5,             /* an NCCL call failed                       */
  FNO_ERR_WORKSPACE = 6         /* workspace too small or misaligned         */
} fno_status;

/* flags (fno_problem.flags) */
#define FNO_ACT_GELU 0u         /* sigma = GELU, exact erf form (default; Q6) */
#define FNO_ACT_NONE 1u         /* sigma = identity                          */

typedef struct fno_comm_s* fno_comm_t;
typedef struct fno_plan_s* fno_plan_t;

/* The problem statement of the paper (P:52 modes per dimension, P:182 grid
 * shape, P:183 width, P:61/P:185 worker partition). */
typedef struct {
  int64_t grid[4];   /* global X, Y, Z, T                                     */
  int32_t batch;     /* B >= 1                                                */
  int32_t width;     /* C = C_in = C_out >= 1                                 */
  int32_t modes[4];  /* mx, my, mz (keep {0..m-1} ∪ {n-m..n-1}, 2m <= n);
                        mt (keep {0..mt-1}, mt <= T/2 + 1)                    */
  int32_t pgrid[2];  /* px, py: x/y worker grid; z, t undecomposed            */
  uint32_t flags;    /* FNO_ACT_*                                             */
} fno_problem;

/* ---- communicator (NCCL over NVLink/NVSwitch) ---------------------------- */
/* Rank 0 creates the 128-byte unique id; the caller broadcasts it (e.g. with
 * torch.distributed) and every rank calls fno_comm_init with its rank and the
 * device it has made current.  Returns FNO_ERR_NCCL on NCCL failure. */
fno_status fno_comm_unique_id(uint8_t id[128]);
fno_status fno_comm_init(const uint8_t id[128], int nranks, int rank, fno_comm_t* comm);
/* A communicator descriptor without a transport: plans built on it answer the
 * host-side queries (boxes, owned modes, workspace size) for rank `rank` of
 * `nranks` without any GPU; compute calls on such a plan with P > 1 return
 * FNO_ERR_INVALID_STATE. */
fno_status fno_comm_init_local(int nranks, int rank, fno_comm_t* comm);
fno_status fno_comm_destroy(fno_comm_t comm);
fno_status fno_comm_size(fno_comm_t comm, int* nranks, int* rank);

/* ---- plan ---------------------------------------------------------------- */
/* Validates the problem (grid, width > 0; 2m <= n on x, y, z; 1 <= mt <=
 * T/2+1; px*py == comm size (comm may be NULL iff px*py == 1); X % px == 0 and
 * Y % py == 0) and derives the local box, the kz ownership block and the
 * workspace layout.  FNO_ERR_INVALID_ARGUMENT on a bad problem; FNO_ERR_PLAN if
 * the transform sizes are outside what the kernels support (any length whose
 * prime factors are 2, 3, 5 up to 1024 per axis). */
fno_status fno_plan_create(const fno_problem* problem, fno_comm_t comm, fno_plan_t* plan);
fno_status fno_plan_destroy(fno_plan_t plan);
/* Bytes of device workspace the caller must provide (256-byte aligned). */
fno_status fno_plan_workspace_size(fno_plan_t plan, size_t* bytes);
fno_status fno_plan_set_workspace(fno_plan_t plan, void* dptr, size_t bytes);
/* Collective (every rank of the plan's communicator calls it, after
 * fno_plan_set_workspace): maps every rank's workspace into this process with
 * CUDA IPC over NVLink, so that the pencil repartitions become
 * direct peer stores -- pass A writes its retained-mode slab straight into the
 * kz owners' receive buffers and the y-inverse writes straight into the x/y
 * owners' receive buffers -- and each exchange reduces to a barrier (a one-int
 * NCCL all-reduce).  Only the retained-mode slab crosses NVLink, as before.
 * Stream-ordered on `stream` (synchronised once inside).  No-op when P == 1.
 * The workspace must stay allocated for the plan's lifetime, and
 * fno_plan_set_workspace / fno_plan_set_io_partition are rejected
 * (FNO_ERR_INVALID_STATE) once the peers are connected; the mappings are closed
 * by fno_plan_destroy.  The choice is collective: if any rank cannot export its
 * workspace or open a peer's (CUDA IPC refused, no peer access, ...), every rank
 * returns FNO_OK and keeps the NCCL send/recv exchanges (query with
 * fno_plan_peer_enabled).  FNO_ERR_CUDA / FNO_ERR_NCCL only when the handle
 * all-gather itself fails. */
fno_status fno_plan_connect_peers(fno_plan_t plan, void* stream);
/* Which pass C kernel the plan launches for mode 0 (spectral u), 1 (layer
 * forward), 2 (layer backward): info = {family, padded width, input-ring
 * stages / tile buffers, dynamic shared memory bytes}; family 4 = the
 * warp-specialised tcgen05 kernel (pass_c4), 3 = pass_c3, 2 = pass_c2 (FFMA),
 * 1 = the generic pass_c; 5 (mode 2 only, C <= 20) = the split backward: dv =
 * W^T dz + S^T dz by the mode-1 family's kernel run with W^T, no bias and the
 * identity (info describes that kernel), then dW and db by the streaming
 * dw_partial kernel over dz and v (8 B per point-channel, fixed-order sums).
 * The family-4 launch falls back to the next family when the tensors'
 * alignment rules out its TMA view. */
fno_status fno_plan_pass_c_info(fno_plan_t plan, int mode, int64_t info[4]);
/* Selects the pass C kernel family (as in fno_plan_pass_c_info) for mode 0
 * (spectral u), 1 (layer forward) or 2 (layer backward).  fno_plan_create
 * picks the measured-fastest eligible family; this call is for A/B runs and
 * tests.  FNO_ERR_PLAN if the family does not cover the problem. */
fno_status fno_plan_set_pass_c(fno_plan_t plan, int mode, int family);
/* *enabled = 1 if fno_plan_connect_peers switched the exchanges to peer stores. */
fno_status fno_plan_peer_enabled(fno_plan_t plan, int* enabled);
/* Caller-side partition of the fields (the paper's App. A 3-D
 * spatial and temporal partitions): io_pgrid = (px', py', pz', pt')
 * over the same P ranks (row-major, each extent divisible by its part).  The
 * compute calls then take and return v, y, u, g, dy, dv in that partition
 * (this rank's box: fno_plan_io_box) and repartition them to and from the
 * plan's x/y grid around the layer ("a repartition operator is used to
 * take the data to a partition of only the x and y dimensions"; two extra
 * all-to-alls of the full field per call, generalised R_{P->Q}).  z_save
 * / z_saved stay in the x/y layout (an opaque buffer of the same size).  Must be
 * called before fno_plan_workspace_size / fno_plan_set_workspace (the workspace
 * grows by three field buffers and the repartition scratch).  The network calls
 * (fno_net_*) keep the x/y partition.  (px, py, 1, 1) is the plan's own grid:
 * no-op. */
fno_status fno_plan_set_io_partition(fno_plan_t plan, const int32_t io_pgrid[4]);
/* This rank's box of the io partition: [lo, hi) per X, Y, Z, T. */
fno_status fno_plan_io_box(fno_plan_t plan, int64_t lo[4], int64_t hi[4]);
/* Local x/y box of this rank in global coordinates: [lo, hi) per X, Y, Z, T. */
fno_status fno_plan_local_box(fno_plan_t plan, int64_t lo[4], int64_t hi[4]);
/* Retained-kz index block [kz_lo, kz_hi) whose weights this rank owns after the
 * forward exchange (only owners apply R_phi).  May be empty. */
fno_status fno_plan_owned_modes(fno_plan_t plan, int32_t* kz_lo, int32_t* kz_hi);
/* Number of complex elements of V^ saved by the forward for the backward:
 * [B][C][2mx][2my][kz_hi-kz_lo][mt]. */
fno_status fno_plan_vhat_elems(fno_plan_t plan, size_t* elems);

/* ---- spectral convolution S (Eq. 3 / Eq. sconv_dist) ---------------------- */
/* u = S v.  v, u: float [B][C][Xl][Yl][Z][T]; R: float2 [C][C][2mx][2my][nkz][mt].
 * vhat_save (nullable): float2 [B][C][2mx][2my][nkz][mt] receives V^ = F v on
 * the owned modes. */
fno_status fno_spectral_conv_fwd(fno_plan_t plan, const float* v, const void* R, float* u,
                                 void* vhat_save, void* stream);
/* Adjoint: dv = S^T g (S with R^H[i,o,k] = conj R[o,i,k]) and, if dR != NULL,
 * the weight gradient dR[i,o,k] (+)= (c(kt)/N) sum_b conj(V^[b,i,k]) G^[b,o,k]
 * with G^ = F g (requires vhat_saved).  dv may be NULL.  accumulate: 0
 * overwrites dR, 1 adds into it. */
fno_status fno_spectral_conv_bwd(fno_plan_t plan, const float* g, const void* R, const void* vhat_saved,
                                 float* dv, void* dR, int accumulate, void* stream);

/* ---- DFNO block (Eq. dist_block) ----------------------------------------- */
/* z = W v + b + S v ; y = sigma(z).  z_save, vhat_save nullable (training
 * mode stores them for fno_layer_bwd). */
fno_status fno_layer_fwd(fno_plan_t plan, const float* v, const void* R, const float* W, const float* b,
                         float* y, float* z_save, void* vhat_save, void* stream);
/* Backward of the block given dy: dz = dy sigma'(z); dv = W^T dz + S^T dz;
 * dW[o,i] (+)= sum dz[o] v[i]; db[o] (+)= sum dz[o] (both already summed over
 * all ranks in ascending rank order: the broadcast adjoint);
 * dR as in fno_spectral_conv_bwd.  db may be NULL. */
fno_status fno_layer_bwd(fno_plan_t plan, const float* v, const float* z_saved, const void* vhat_saved,
                         const float* dy, const void* R, const float* W, float* dv, void* dR,
                         float* dW, float* db, int accumulate, void* stream);

/* ---- whole network (PAPER.md "Full Network") ---- */
/*   a1   = W_t a + b_t            time affine, input a has a time axis of size 1
 *   nu_0 = W_c a1 + b_c           channel affine C_in -> C
 *   nu_{k+1} = sigma(W nu_k + S nu_k), k < K, no sigma after the last block       P:161-166 (N1b)
 *   u    = W_p nu_K (+ b_p)       projection C -> 1                                P:171-173 (N1c)
 *   L    = ||u - y||_2 / ||y||_2  relative L2 misfit over all ranks
 * All pointers are device pointers on the plan's device, caller-owned; shapes
 * use the plan's local box: a [B][C_in][Xl][Yl][Z] (the size-1 time axis
 * dropped), nu / z / scratch [B][C][Xl][Yl][Z][T], u / y [B][1][Xl][Yl][Z][T].
 * The calls are stream-ordered and, for P > 1, collective (W_t, b_t, W_c, b_c,
 * W_p, b_p are replicated; their gradients come back summed over ranks in rank
 * order, the broadcast adjoint P:64; R is kz-owned as in fno_layer_*). */
#define FNO_NET_MAXK 16
typedef struct {
  int32_t layers;       /* K, 1 <= K <= FNO_NET_MAXK */
  int32_t in_channels;  /* C_in, 1..4 (2 in the paper's CO2 example) */
  int32_t proj_bias;    /* 1: u = W_p nu_K + b_p; 0: no projection bias */
} fno_net_desc;
typedef struct {
  float* Wt;                   /* [T]  (W_t is T x 1) */
  float* bt;                   /* [T] */
  float* Wc;                   /* [C][C_in] */
  float* bc;                   /* [C] */
  void* R[FNO_NET_MAXK];       /* float2 [C][C][2mx][2my][nkz][mt] per block */
  float* W[FNO_NET_MAXK];      /* [C][C] (C_out, C_in) per block */
  float* b[FNO_NET_MAXK];      /* [C] per block */
  float* Wp;                   /* [C] */
  float* bp;                   /* [1]; unused when proj_bias == 0 */
} fno_net_params;              /* also the layout of the gradients */
typedef struct {
  float* nu[FNO_NET_MAXK + 1]; /* nu_0 .. nu_K, written by fno_net_fwd */
  float* z[FNO_NET_MAXK];      /* pre-activations of blocks 0 .. K-2 (block K-1 has none) */
  void* vhat[FNO_NET_MAXK];    /* V^ per block, fno_plan_vhat_elems complex each */
} fno_net_acts;
/* Bytes of device scratch ("net workspace") fno_net_loss / fno_net_bwd need. */
fno_status fno_net_workspace_size(fno_plan_t plan, const fno_net_desc* desc, size_t* bytes);
/* Forward: lift, the K blocks (training mode: z and V^ kept), projection. */
fno_status fno_net_fwd(fno_plan_t plan, const fno_net_desc* desc, const fno_net_params* params, const float* a,
                       const fno_net_acts* acts, float* u, void* stream);
/* loss3 (device, 3 floats) = {L, ||u - y||^2, ||y||^2} over all ranks (fp64
 * partial sums in a fixed order); the fp64 sums stay in net_ws for fno_net_bwd. */
fno_status fno_net_loss(fno_plan_t plan, const float* u, const float* y, float* loss3, void* net_ws, void* stream);
/* Backward of L through projection, blocks and lift (after fno_net_loss on the
 * same u, y and net_ws).  grads: same layout as params (grads->bp ignored when
 * proj_bias == 0); every gradient is overwritten.  scratch0 / scratch1: two
 * field buffers for the adjoint ping-pong. */
fno_status fno_net_bwd(fno_plan_t plan, const fno_net_desc* desc, const fno_net_params* params, const float* a,
                       const fno_net_acts* acts, const float* u, const float* y, const fno_net_params* grads,
                       float* scratch0, float* scratch1, void* net_ws, void* stream);
/* Data x domain hybrid: in-place NCCL all-reduce of n floats over
 * the ranks of comm -- the replicas of a domain-decomposed network that hold the
 * same x/y box of different samples -- summed (average = 0) or averaged
 * (average = 1), e.g. the gradients after fno_net_bwd.  Stream-ordered, collective. */
fno_status fno_comm_allreduce(fno_comm_t comm, float* buf, size_t n, int average, void* stream);
/* One Adam step (Kingma & Ba, bias-corrected; P:187 uses lr 1e-3) on n floats:
 * m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2; p -= lr (m/(1-b1^step)) /
 * (sqrt(v/(1-b2^step)) + eps).  Complex R is passed as 2n floats (real and
 * imaginary parts updated independently, reading N1d).  step >= 1. */
fno_status fno_adam(float* p, const float* g, float* m, float* v, size_t n, float lr, float beta1, float beta2,
                    float eps, int step, void* stream);

/* ---- repartition R_{P->Q} -------------------------------------- */
/* Moves a tensor of `ndim` <= 8 dimensions and global shape `global_shape`
 * from the Cartesian partition src_pgrid to dst_pgrid over the ranks of comm
 * (row-major ranks, balanced blocks: first n mod p blocks one longer).  Both
 * partitions must have exactly comm-size workers.  src_local / dst_local are
 * this rank's boxes (contiguous, row-major, elem_bytes per element).
 * Workspace: query with workspace == NULL -> *ws_bytes receives the size. The
 * adjoint is the same call with the pgrids swapped. */
fno_status fno_repartition(fno_comm_t comm, int ndim, const int64_t* global_shape, const int32_t* src_pgrid,
                           const int32_t* dst_pgrid, size_t elem_bytes, const void* src_local, void* dst_local,
                           void* workspace, size_t* ws_bytes, void* stream);

/* ---- plan groups: a P-rank decomposition in ONE process on ONE device ------ */
/* The decomposed data path of Eq. sconv_dist without P GPUs: plan
 * r (r = 0..n-1) is rank r of the same n-rank problem, created on a
 * fno_comm_init_local(n, r) communicator, its workspace set on the common
 * device.  fno_group_connect points every plan's exchange destinations at the
 * other plans' workspaces (the peer-store exchange of fno_plan_connect_peers
 * with same-device pointers), after which the plans are usable only through
 * the fno_group_* calls.  Each group call runs one stage for every rank before
 * the next stage (pass A of all ranks, then pass B, then pass C, then the
 * rank-ordered dW / db sum), all on `stream`, so stream order is the exchange
 * barrier and no rank ever waits for another.  Arrays hold one pointer per
 * rank (the rank's local box / kz block, as in the per-plan calls; vhat_save
 * entries and the vhat_save / z_save / dv / dR arrays themselves nullable as
 * in the per-plan calls); W, b, dW, db are single (replicated) tensors and dW
 * / db come back summed over the ranks in rank order.  Errors as in the
 * per-plan calls; FNO_ERR_INVALID_STATE for plans that are not a connected
 * group in rank order. */
fno_status fno_group_connect(int n, fno_plan_t* plans);
fno_status fno_group_spectral_conv_fwd(int n, fno_plan_t* plans, const float* const* v, const void* const* R,
                                       float* const* u, void* const* vhat_save, void* stream);
fno_status fno_group_spectral_conv_bwd(int n, fno_plan_t* plans, const float* const* g, const void* const* R,
                                       const void* const* vhat_saved, float* const* dv, void* const* dR,
                                       int accumulate, void* stream);
fno_status fno_group_layer_fwd(int n, fno_plan_t* plans, const float* const* v, const void* const* R, const float* W,
                               const float* b, float* const* y, float* const* z_save, void* const* vhat_save,
                               void* stream);
fno_status fno_group_layer_bwd(int n, fno_plan_t* plans, const float* const* v, const float* const* z_saved,
                               const void* const* vhat_saved, const float* const* dy, const void* const* R,
                               const float* W, float* const* dv, void* const* dR, float* dW, float* db,
                               int accumulate, void* stream);

/* ---- instrumentation ------------------------------------------------------ */
/* When enabled, every stage of every call on this plan (pass A, exchange 1,
 * the pass-B kernels, mixing, exchange 2, pass C, the dW reduction) is
 * bracketed by CUDA events recorded on the call's stream (CUDA
 * events per stage).  fno_plan_profile_read waits for the recorded events and
 * returns, per stage i < fno_profile_stage_count(), the summed milliseconds and
 * the number of timed launches since the last read; then it resets.  nstages
 * must be >= fno_profile_stage_count(). */
fno_status fno_plan_profile_enable(fno_plan_t plan, int enable);
fno_status fno_plan_profile_read(fno_plan_t plan, double* ms, int64_t* count, int nstages);
int fno_profile_stage_count(void);
const char* fno_profile_stage_name(int stage);
/* Number of kernels this process has launched through libfno (NCCL's own
 * kernels are not counted). */
unsigned long long fno_kernel_launches(void);

const char* fno_status_string(fno_status s);
const char* fno_last_error(void);
int fno_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FNO_H_ */
