/*
 * parrot_b200.h -- C ABI of libparrot_b200.so, the B200 (sm_100a) device-side
 * hot path of FedML Parrot's simulator.
 *
 * The reference (FedML Parrot, `fedsim` 0.1.0, pure Python/NumPy) has no FFI:
 * its "plugin" boundary is the in-process Python API.  Each
 * entry point below names the reference function it replaces; the Python
 * package `paper_2303_01778_b200` binds them through ctypes and presents the
 * reference's own API (client_execute / local_fold / global_fold /
 * server_update / StateStore / schedule / DeviceWorker.execute_clients).
 *
 * Conventions
 *  - All buffers are caller-owned device pointers (unless marked HOST); the
 *    library never allocates on the hot path.  `stream` is a cudaStream_t
 *    passed as void*; every kernel is asynchronous on it.
 *  - Return 0 on success, a PB_ERR_* code otherwise; pb_last_error() returns
 *    the thread-local message of the last failure.
 *  - Parameter vectors are flat fp32 in the model's canonical order.  A
 *    "group" is G clients laid out as rows of a [G, stride] matrix.
 */
#ifndef PARROT_B200_H
#define PARROT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PB_OK 0
#define PB_ERR_INVALID 1   /* bad argument / unsupported shape  */
#define PB_ERR_CUDA 2      /* CUDA runtime error                */

const char* pb_last_error(void);
int pb_version(void);
int pb_device_sm_count(int device);
/* sizeof of the argument structs, so bindings can check their layout:
 * out[0] pb_lr_train_args, out[1] pb_cnn_train_args, out[2]
 * pb_cnn_lazy_fold_args, out[3] pb_resnet_train_args; returns how many it
 * wrote (min(n, 4)). */
int pb_abi_sizes(int64_t* out, int n);

/* Launch accounting and optional per-kernel-class timing (CUDA events on the
 * launching stream).  pb_launch_count: kernels launched by this library so far.
 * pb_prof_collect fills ms[id] / count[id] for the kernel classes
 *   0 fold1 1 fold_group 2 lincomb 3 delta_affine 4 state_gather
 *   5 state_scatter 6 lr_train 7 lr_eval 8 cnn_slots 9 cnn_fwd 10 cnn_fc1_fwd
 *   11 cnn_head 12 cnn_fc1_bwd 13 cnn_bwd_conv 14 cnn_wgrad 15 cnn_lz_xt
 *   16 cnn_lz_gram_fwd 17 cnn_lz_fwd 18 cnn_lz_gram_bwd 19 cnn_lz_bwd 20 cnn_lz_mat
 *   21 rn_conv_fwd 22 rn_conv_dgrad 23 rn_conv_wgrad 24 rn_norm 25 rn_head 26 rn_sgd
 * recorded since the last collect (nslots >= 27), synchronising on them. */
int pb_prof_enable(int on);
/* Restrict profiling to the kernel classes whose bit (1 << class id) is set
 * (default: all).  Each recorded launch adds two CUDA events to the stream. */
int pb_prof_select(uint64_t mask);
int64_t pb_launch_count(void);
int pb_prof_collect(double* ms, int64_t* count, int nslots);

/* ---------------------------------------------------------------------------
 * Host-side scheduling / RNG (native runtime around the kernels)
 * ------------------------------------------------------------------------- */

/* Greedy min-makespan assignment.  Replaces fedsim/schedule.py:88-126
 * (_greedy_jit, the numba kernel) and :48-85 (_greedy_core).  sizes_desc are
 * task sizes already sorted largest-first; assign[i] receives the device of
 * task i, loads[k] the predicted load of device k.  HOST pointers.  Compiled
 * with -ffp-contract=off: bit-identical to the reference. */
int pb_greedy_assign(const double* sizes_desc, int64_t n, const double* t, const double* b,
                     int64_t k, int64_t* assign, double* loads);

/* Per-client minibatch orders.  Replaces the per-epoch
 * `default_rng([seed, 6, client, round]).permutation(n)` of
 * fedsim/trainer.py:445,452-453 (NumPy PCG64 + SeedSequence + Fisher-Yates
 * with masked rejection, restated bit-exactly).  For client i the output
 * out[offset[i] + e*n[i] + j] = row_base[i] + perm_e[j], e < epochs.
 * keys is [g][4] = (seed, stream, client_id, round).  HOST pointers. */
int pb_minibatch_rows(const uint64_t* keys, const int64_t* n, const int64_t* offset,
                      const int64_t* row_base, int64_t g, int epochs, int32_t* out,
                      int threads);

/* ---------------------------------------------------------------------------
 * (b) fused weighted fold  -- fedsim/aggregate.py:76-102 (local_fold) and
 *     :130-142 (global_fold's device-order sum)
 * ------------------------------------------------------------------------- */

/* acc[i] = fma(w, x[i], acc[i]) -- one client folded into a running sum. */
int pb_fold_f32(float* acc, const float* x, float w, int64_t n, void* stream);

/* acc[i] += sum_{j<g} w[j] * xs[order[j]*x_stride + i], j ascending (plan
 * order), one pass over acc.  order may be NULL (identity), w may be NULL
 * (all ones).  The sum is sequential per element, so the result equals g
 * successive pb_fold_f32 calls bit for bit. */
int pb_fold_group_f32(float* acc, const float* xs, int64_t x_stride, const int32_t* order,
                      const float* w, int64_t g, int64_t n, void* stream);

/* out[i] = a*x[i] + b*y[i] + c*z[i]; NULL inputs contribute nothing.  Used by
 * global_fold's final divide and the plugin server rules
 * (fedsim/trainer.py:232-234, :280-285, :340-348, :397-407). */
int pb_lincomb_f32(float* out, const float* x, float a, const float* y, float b,
                   const float* z, float c, int64_t n, void* stream);

/* Plugin finalize (fedsim/trainer.py:268-278, :325-338, :388-395) for a group:
 * out[j,i] = s[j]*(a[j,i] - base[i]) + c*cvec[i] + d*dmat[j,i].
 * cvec/dmat may be NULL. */
int pb_delta_affine_group(float* out, int64_t out_stride, const float* a, int64_t a_stride,
                          const float* base, const float* s, const float* cvec, float c,
                          const float* dmat, int64_t d_stride, float d, int64_t g, int64_t n,
                          void* stream);

/* ---------------------------------------------------------------------------
 * (c) client-state gather / scatter -- fedsim/statestore.py:147-210
 *     (StateStore.load/save) + default_state (fedsim/trainer.py:315-317,
 *     :376-378): gather slot -1 writes the all-zero default state, slot <= -2
 *     leaves the work row alone (the client lives in another tier); scatter
 *     skips slot < 0.  `store` may be an HBM matrix or pinned (device-mapped)
 *     host memory: the host tier of a store larger than its HBM budget is
 *     moved by the same kernels over the host link.
 * ------------------------------------------------------------------------- */
int pb_state_gather(float* work, int64_t work_stride, const float* store, int64_t store_stride,
                    const int32_t* slot, int64_t g, int64_t width, void* stream);
int pb_state_scatter(float* store, int64_t store_stride, const float* work, int64_t work_stride,
                     const int32_t* slot, int64_t g, int64_t width, void* stream);

/* ---------------------------------------------------------------------------
 * (a) batched client training, multinomial logistic regression
 *     -- fedsim/trainer.py:427-477 (client_execute) with the plugin
 *     local_gradient hooks (:223, :249-257, :319-323, :380-386) fused in:
 *     grad = CE grad + mu*(w - w0) + cg*ctrl_g + cc*ctrl_c[client]
 * One CTA per client; the whole local run (E epochs x ceil(n/bs) steps) stays
 * on chip.  w layout: W[C][F] row-major then b[C].
 * ------------------------------------------------------------------------- */
typedef struct {
  const float* X;          /* [rows, F] fp32, all clients packed           */
  const int32_t* Y;        /* [rows] labels                                 */
  const int32_t* order;    /* packed minibatch row ids (pb_minibatch_rows)  */
  const int64_t* order_off;/* [g] offset of client j's rows in `order`      */
  const int32_t* n;        /* [g] samples per client                        */
  const float* w0;         /* [P] start model (the global bundle)           */
  float* w_out;            /* [g, P] end model per client                   */
  const float* ctrl_g;     /* [P] shared correction or NULL                 */
  const float* ctrl_c;     /* [g, ctrl_stride] per-client correction / NULL */
  int64_t ctrl_stride;
  double* loss_sum;        /* [g] sum of per-step losses                    */
  int32_t* steps;          /* [g] steps taken                               */
  int32_t* nonfinite;      /* [g] first step whose loss was not finite, -1  */
  int64_t g;
  int32_t F, C, epochs, batch_size;
  float lr, mu, prox_loss, cg, cc;
  int64_t* client_ns;      /* [g, 2] %globaltimer at the client's first and  */
                           /* last instruction (real-clock records) or NULL  */
} pb_lr_train_args;
int pb_lr_train_group(const pb_lr_train_args* args, void* stream);

/* evaluate (fedsim/trainer.py:148-158): out2[0] += #correct, out2[1] += sum CE */
int pb_lr_eval(const float* X, const int32_t* Y, int64_t rows, int F, int C, const float* w,
               double* out2, void* stream);

/* ---------------------------------------------------------------------------
 * (a) batched client training, 2-layer FEMNIST CNN (BASELINE config 2; the
 *     reference has no CNN -- semantics follow client_execute,
 *     fedsim/trainer.py:427-477).  Parameters: flat fp32 per client in the
 *     layout of models.py:cnn_spec.  All active clients advance one SGD step
 *     per sweep; conv2 forward/dgrad/wgrad run on tcgen05 (bf16 operands,
 *     fp32 TMEM accumulation), the rest in fp32.  Workspace buffers are
 *     caller-allocated, sized per slot (= client) for BS samples:
 *       ws_slots 32 B, ws_p1 BS*21568 B, ws_am1 BS*6272 B, ws_p2 BS*3136 f32,
 *       ws_am2 BS*3136 B, ws_h/ws_dh BS*512 f32, ws_dp2 BS*3136 f32,
 *       ws_dz BS*43136 B, ws_dp1 BS*6272 f32 (per-sample conv1/bias gradient
 *       partials, 896 used), ws_dht 16384 f32 per slot.
 * ------------------------------------------------------------------------- */
typedef struct {
  const float* X;           /* [rows, 784] fp32 images                        */
  const int32_t* Y;         /* [rows] labels                                  */
  const int32_t* order;     /* packed minibatch row ids                       */
  const int64_t* order_off; /* [g] per client                                 */
  const int32_t* n;         /* [g] samples per client                         */
  const int32_t* rank;      /* [g] slot -> client row, by step count desc     */
  const int32_t* active;    /* HOST [sweeps]: clients still stepping per sweep*/
  int32_t sweeps;
  float* w;                 /* [g, w_stride] params (start = w0), in place    */
  int64_t w_stride;         /* row stride of w in floats, multiple of 4       */
  const float* w0;          /* [P]                                            */
  const float* ctrl_g;      /* [P] or NULL                                    */
  const float* ctrl_c;      /* [g, ctrl_stride] or NULL                       */
  int64_t ctrl_stride;
  double* loss_sum;         /* [g] (zero-initialised by the caller)           */
  int32_t* steps;           /* [g] (zero-initialised)                         */
  int32_t* bad;             /* [g] (-1 initialised): step of a non-finite loss*/
  void* ws_slots;
  uint8_t* ws_p1;
  uint8_t* ws_am1;
  float* ws_p2;
  uint8_t* ws_am2;
  float* ws_h;
  float* ws_dh;
  float* ws_dp2;
  uint8_t* ws_dz;
  float* ws_dp1;
  float* ws_dht;            /* per slot: 512*32 f32 (dH transposed, zero-padded) */
  /* Low-rank fc1 for plain SGD (mu = 0, no control variates); all NULL for
   * the direct per-client fc1.  The history and W0 copies are bf16 (the
   * tensor-core operands, rounded to nearest once when written).  Client row
   * r owns history rows [lz_hoff[r], lz_hoff[r] + lz_hlen[r]) of lz_rows,
   * lz_hlen[r] = round_up(steps_r*BS, 64);
   * step t's sample i is row t*BS + i.  Every client's fc1 weights stay
   * W0 - lr * sum_t dH_t^T X_t during the round (never materialised per
   * step); they are written to w once, after the last sweep.  The history
   * GEMMs read whole 32-row chunks and multiply the rows a client has not
   * written by exact zeros (the kernels zero each client's dH^T pad
   * columns), so the four history buffers need only hold FINITE values on
   * entry (zero them once after allocation or after a diverged client). */
  void* lz_hx;              /* [lz_rows, 3136] bf16                           */
  void* lz_hxt;             /* unused (the GEMMs over history rows read lz_hx */
                            /* MN-major); may be NULL                         */
  void* lz_hd;              /* [lz_rows, 512] bf16                            */
  void* lz_hdt;             /* unused (history rows are read MN-major); NULL  */
  const int64_t* lz_hoff;   /* [g]                                            */
  const int32_t* lz_hlen;   /* [g]                                            */
  void* lz_w0t;             /* 2*3136*512 bf16 scratch: W1 of w0 transposed,  */
                            /* then as is                                     */
  float* lz_zp;             /* max_t active_t*njt_t * 512*32 f32, njt_t = ceil(t*BS/128) */
  void* lz_gdt;             /* max_t active_t*njt_t * 32*128 bf16             */
  float* lz_fpart;          /* max(74, g)*512*32 f32: forward GEMM partials   */
  int64_t lz_rows;          /* total history rows (multiple of 64)            */
  int32_t lz_defer;         /* 1: leave the fc1 block of w unmaterialised      */
                            /*    (fold it with pb_cnn_lazy_fold instead)      */
  int32_t lz_switch;        /* > 0: from sweep lz_switch on, the clients still */
                            /* stepping (more than lz_switch steps) leave the  */
                            /* low-rank form: their fc1 is materialised once   */
                            /* and trained by the direct kernels (the history */
                            /* re-read grows with the step count).  Their w   */
                            /* rows hold the final fc1 even with lz_defer.    */
  int64_t g;
  int32_t C, BS, batch_size, epochs, samples_per_cta;
  float lr, mu, cg, cc;
  int64_t* timeline;        /* [sweeps + 1] %globaltimer at the start of each */
                            /* sweep and after the last one, or NULL: sweep s */
                            /* lasts timeline[s+1] - timeline[s] ns and is    */
                            /* shared by its active clients (real clock)      */
  void* ws_w2b;             /* [g][102400 B] scratch: bf16 conv2 weights in   */
                            /* the tensor-core layout, rebuilt from w at the  */
                            /* start of a call and kept in step with it       */
} pb_cnn_train_args;
int pb_cnn_train_group(const pb_cnn_train_args* args, void* stream);

/* Deferred fc1 fold of a low-rank CNN round (local_fold, fedsim/aggregate.py
 * :76-102, for the fc1_w entry of a FedAvg device partial):
 *   acc += wsum * W0 - lr * sum_j w_j * HD_j^T HX_j
 * over the device's clients j, whose history rows are [row_lo, row_hi) of
 * the round's [lz_rows] history (pb_cnn_train_group with lz_defer = 1).
 * The weighted dH rows w_j * dH_j are split into two bf16 terms (high part
 * in hd in place -- round scratch --, low part in hd_lo), so the
 * weighting is exact to ~2^-17 and both terms run on bf16 tensor cores.
 * part: splits * 512 * 3136 f32 scratch. */
typedef struct {
  float* acc;               /* [512*3136] fc1_w accumulator of the partial     */
  const float* w0;          /* [P] round-start model                           */
  const void* hx;           /* [hrows, 3136] bf16: the X history              */
  void* hd;                 /* [hrows, 512] bf16 (overwritten: w_j * dH, high) */
  int64_t hrows, row_lo, row_hi;
  const int64_t* hoff;      /* [nclients] first history row of each client    */
  const int32_t* nrows;     /* [nclients] live history rows (steps * BS)       */
  const float* w;           /* [nclients] fold weights (sample counts)         */
  int64_t nclients;
  float* part;
  int32_t splits;
  float wsum, lr;
  void* hd_lo;              /* [hrows, 512] bf16 scratch: w_j * dH, low part   */
} pb_cnn_lazy_fold_args;
int pb_cnn_lazy_fold(const pb_cnn_lazy_fold_args* args, void* stream);

/* Forward-only evaluation of parameter row 0 of args->w on `rows` samples
 * (order = row ids); out2[0] += #correct, out2[1] += sum CE.  args->g is the
 * workspace capacity in slots of BS samples. */
int pb_cnn_eval(const pb_cnn_train_args* args, int64_t rows, double* out2, void* stream);

/* ---------------------------------------------------------------------------
 * (a) batched client training, ResNet-18 with GroupNorm (BASELINE config 4;
 *     the reference has no ResNet -- semantics follow client_execute,
 *     fedsim/trainer.py:427-477, plain SGD / FedAvg).  Parameters: flat fp32
 *     per client in the layout of models.py:resnet_layout (P = 11,173,962 at
 *     C = 10); inputs 3072 fp32 = a 32x32x3 NHWC image.  All active clients
 *     advance one SGD step per sweep; every convolution (forward, dgrad,
 *     wgrad) is a tcgen05 implicit GEMM on bf16 operands with fp32 TMEM
 *     accumulation.  Workspaces are caller-allocated; their per-slot sizes
 *     come from pb_resnet_workspace(BS, C, out4):
 *       out4[0] arena bytes per slot, out4[1] P16 (bf16 weight-copy row
 *       length), out4[2] wgrad-partial floats per slot, out4[3] GroupNorm
 *       partial floats per slot.
 * ------------------------------------------------------------------------- */
typedef struct {
  const float* X;           /* [rows, 3072] fp32 images                       */
  const int32_t* Y;         /* [rows] labels                                  */
  const int32_t* order;     /* packed minibatch row ids (pb_minibatch_rows)   */
  const int64_t* order_off; /* [g] per client                                 */
  const int32_t* n;         /* [g] samples per client                         */
  const int32_t* rank;      /* [g] slot -> client row, by step count desc     */
  const int32_t* active;    /* HOST [sweeps]: clients still stepping per sweep*/
  int32_t sweeps;
  float* w;                 /* [g, w_stride] params (start = w0), in place    */
  int64_t w_stride;         /* floats, multiple of 4, >= P                    */
  double* loss_sum;         /* [g] (zero-initialised by the caller)           */
  int32_t* steps;           /* [g] (zero-initialised)                         */
  int32_t* bad;             /* [g] (-1 initialised)                           */
  void* ws_slots;           /* 16 B per slot                                  */
  void* ws_w16;             /* [g][P16] bf16                                  */
  uint8_t* ws_arena;        /* [g][arena bytes]                               */
  float* ws_part;           /* [g][partial floats]                            */
  float* ws_gnp;            /* [g][GroupNorm partial floats]                  */
  int64_t g;
  int32_t C, BS, batch_size, epochs;
  float lr;
  int64_t* timeline;        /* [sweeps + 1] sweep start stamps, as for the CNN */
  /* Plugin terms of the local gradient, as for the CNN (fedsim/trainer.py
   * :237-257 FedProx, :288-348 SCAFFOLD): every SGD step uses
   *   g + mu * (w - w0) + cg * ctrl_g + cc * ctrl_c[client row]
   * (all terms off: mu = 0, ctrl_g = ctrl_c = NULL -- FedAvg / FedNova).     */
  const float* w0;          /* [P] round-start model (FedProx)                */
  const float* ctrl_g;      /* [P] or NULL (SCAFFOLD server control)          */
  const float* ctrl_c;      /* [g, ctrl_stride] or NULL (client controls)     */
  int64_t ctrl_stride;
  float mu, cg, cc;
} pb_resnet_train_args;
int pb_resnet_workspace(int BS, int C, int64_t* out4);
int pb_resnet_train_group(const pb_resnet_train_args* args, void* stream);
/* Forward-only evaluation of parameter row 0 of args->w on `rows` samples
 * (order = row ids); out2[0] += #correct, out2[1] += sum CE.  args->g is the
 * workspace capacity in slots of BS samples. */
int pb_resnet_eval(const pb_resnet_train_args* args, int64_t rows, double* out2, void* stream);

/* ---------------------------------------------------------------------------
 * Diagnostics
 * ------------------------------------------------------------------------- */
/* One M x N x K bf16 tcgen05 GEMM D = A * B^T (A [M,K], B [N,K] row-major
 * bf16; D [128,N] fp32 receives all 128 TMEM lanes) through the canonical
 * SWIZZLE_NONE shared-memory layouts; *_mode: 0 K-major, 1 MN-major,
 * 2 K-major "planes" starting `shift` rows in.  Pins the descriptor
 * conventions the conv kernels use (tests only). */
int pb_umma_selftest(const void* A, const void* B, float* D, int M, int N, int K, int a_mode,
                     int b_mode, int shift, void* stream);

/* One ResNet convolution through k_rn_conv (mode 0 fwd, 1 dgrad, 2 wgrad)
 * on caller data, single slot of BS samples of which cnt are live (tests
 * only; allocates scratch).  See csrc/resnet.cu for the layouts. */
int pb_rn_conv_selftest(int mode, int BS, int cnt, int Cinp, int Cout, int H, int R, int stride,
                        const void* x, const void* w, const void* dz, float* out, void* stream);

/* 128 x N x K tf32 GEMM D = A * B^T (A [128,K], B [N,K] row-major fp32) with
 * both operands loaded by TMA into SWIZZLE_128B K-major tiles (tma.cuh
 * conventions; tests only).  N % 16 == 0, N <= 256, K % 32 == 0. */
int pb_tma_tf32_selftest(const float* A, const float* B, float* D, int N, int K, void* stream);

/* D[128][N] = A^T B for bf16 A [K][128], B [K][N] (row-major, MN contiguous)
 * loaded by TMA as MN-major SWIZZLE_128B tiles; lbo/sbo are the descriptor
 * byte offsets under test (tests only).  N % 64 == 0, K % 64 == 0. */
int pb_tma_bf16_mn_selftest(const void* A, const void* B, float* D, int N, int K, int lbo, int sbo, void* stream);

/* TMA read-bandwidth probe (tools only): `ctas` CTAs stream `nbox` 16 KB
 * boxes each from a [rows, cols] f32 buffer; mode 0 = boxes of 128 rows x
 * 128 B at row pitch cols*4, mode 1 = the same bytes as contiguous tiles. */
int pb_tma_bw_probe(const float* base, int mode, int64_t rows, int64_t cols, int ctas, int nbox,
                    unsigned* sink, void* stream);

/* 128 x N x K tf32 tcgen05 GEMM D = A * B^T from fp32 row-major A [128,K],
 * B [N,K]; a_mn/b_mn select MN-major smem staging (tests only). */
int pb_umma_tf32_selftest(const float* A, const float* B, float* D, int N, int K, int a_mn,
                          int b_mn, void* stream);

/* 128 x 32 x 32 tf32 GEMM with the A operand staged by the layout formula in
 * params[0..9] (device int array; see csrc/umma_selftest.cu) -- probes the
 * MN-major tf32 operand convention (tests only). */
int pb_umma_tf32_probe(const float* A, const float* B, float* D, const int* params, void* stream);

/* Issue `iters` back-to-back M x N x 16 bf16 tcgen05 MMAs from smem operands
 * staged in *_mode layouts (as above), round-robin over `naccum` independent
 * TMEM accumulators, and store the elapsed cycles (one CTA, device pointer).
 * Diagnostic for the UMMA throughput table in DESIGN.md. */
int pb_umma_bench(int M, int N, int a_mode, int b_mode, int iters, int naccum, long long* cycles,
                  void* stream);

/* The same issue loop on `grid` CTAs at once (several per SM): per-CTA
 * elapsed cycles and SM ids (device pointers; tests / DESIGN table only). */
int pb_umma_bench_multi(int M, int N, int iters, int grid, long long* cycles, int* smid, void* stream);
/* The conv kernels' MMA pattern on resident smem operands: `ngroups`
 * accumulators, group g's A start g*a_goff bytes further, 8 K steps of
 * `kstep` (A) / `b_kstep` (B, 0 = kstep) bytes per group, `iters` passes, on `grid` CTAs (diagnostic). */
/* TMEM -> register load throughput: `warps` warps per CTA (148 CTAs) each read
 * `cols` columns of their lane quarter `iters` times (diagnostic). */
int pb_tmem_ld_bench(int warps, int cols, int iters, long long* cycles, float* sink, void* stream);
int pb_umma_bench2(int M, int N, int a_mn, int b_mn, uint32_t a_lbo, uint32_t a_sbo, uint32_t b_lbo, uint32_t b_sbo,
                   uint32_t kstep, int ngroups, uint32_t a_goff, int iters, int grid, long long* cycles,
                   uint32_t b_kstep, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PARROT_B200_H */
