/*
 * xbtile.h -- C ABI of the B200 analog-tile hot path (libxbtile.so).
 *
 * This is the drop-in boundary under the reference's tile API.  Each entry
 * point names the reference interface it replaces (paths relative to
 * /root/reference).  Plain pointers and sizes only; no C++ or torch types.
 *
 *   reference                                            here
 *   ----------------------------------------------------  --------------------------------
 *   AnalogTile(d_out,d_in,settings,seed)  tile.hpp:77     xb_tile_create
 *   AnalogTile::clone                     tile.hpp:91     xb_tile_clone
 *   AnalogTile::forward                   tile.hpp:82     xb_tile_forward      (B samples)
 *   AnalogTile::forward_with_io           tile.hpp:95     xb_tile_forward_io
 *   AnalogTile::forward_noisy             tile.hpp:85     xb_tile_forward_noisy
 *   AnalogTile::backward                  tile.hpp:83     xb_tile_backward
 *   AnalogTile::update                    tile.hpp:84     xb_tile_update       (B sequential updates)
 *   AnalogTile::apply_pulse_trains        tile.hpp:103    xb_tile_apply_trains (packed words)
 *   AnalogTile::get/set_weights           tile.hpp:88-89  xb_tile_get/set_weights
 *   AnalogTile::device()                  tile.hpp:107    xb_tile_get/set_device
 *   AnalogTile::apply_temporal_step       tile.hpp:99     xb_tile_temporal_step
 *   program / drift_to                    inference.hpp:49-57  xb_tile_program / xb_tile_drift_to
 *   calibrate_compensation / factor       inference.hpp:68-70  xb_tile_probe_readout
 *   TransferTile                          compound.hpp:93-131  xb_transfer_*
 *
 * Semantics: a call with B samples is exactly B sequential calls of the
 * reference API on the same (fp32) inputs, in sample order.  The weights of
 * the tile are stationary across the B forwards/backwards of one call; an
 * update call applies its B rank-1 pulsed updates in sample order.
 *
 * Errors: every function returns 0 on success, non-zero on error; the
 * thread-local message (naming the field, like xbarsim::Error) is returned by
 * xb_last_error().  CUDA errors are reported the same way.  A failed call
 * leaves the tile's state (weights, noise counters) as it was; the contents
 * of its output buffers are unspecified.  There is no CPU fallback: without a
 * usable sm_100 device every compute entry fails.
 *
 * Host-buffer entries (no suffix) are synchronous: inputs are borrowed for
 * the duration of the call, outputs are written before return.  *_dev
 * entries take device pointers, run asynchronously on the tile's stream and
 * perform no host synchronisation.
 */
#ifndef XBTILE_H
#define XBTILE_H

#include <stdint.h>

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif
#ifdef __cplusplus
extern "C" {
#endif

#define XB_ABI_VERSION 1

/* proj/include/xbarsim/device.hpp:17 */
enum { XB_CONSTANT_STEP = 0, XB_LINEAR_STEP = 1, XB_SOFT_BOUNDS = 2, XB_EXP_STEP = 3 };
/* proj/include/xbarsim/io.hpp:17 */
enum { XB_NM_NONE = 0, XB_NM_ABS_MAX = 1 };
/* additive (no reference symbol): bound management, default none */
enum { XB_BM_NONE = 0, XB_BM_ITERATIVE = 1 };
/* proj/include/xbarsim/pulsed.hpp:19 */
enum { XB_PULSE_STOCHASTIC = 0, XB_PULSE_DETERMINISTIC = 1 };
/* additive: MVM arithmetic. FP32 = exact fp32 FMA (SIMT); TF32 = one tcgen05
 * kind::tf32 pass; TF32X3 = split-precision 3xTF32 (fp32-level accuracy). */
enum { XB_MVM_FP32 = 0, XB_MVM_TF32 = 1, XB_MVM_TF32X3 = 2 };
/* additive: weight storage.  FP32 = one fp32 per cell; FP32X2 = fp32 plus an
 * fp32 compensation term, pulses added error-free (two-sum), so long runs of
 * tiny steps do not accumulate fp32 rounding (the reference stores fp64);
 * AUTO = FP32X2 when dw_min < 2^-12 max(|w_max|, |w_min|), i.e. a pulse is
 * under ~2048 fp32 ulps of the largest weight (e.g. the "ideal" preset). */
enum { XB_W_AUTO = 0, XB_W_FP32 = 1, XB_W_FP32X2 = 2 };

/* proj/include/xbarsim/device.hpp:24-39 (same fields and defaults) */
typedef struct xb_device_params {
  int32_t kind;
  int32_t _pad;
  double dw_min, dw_min_dtod, dw_min_std, up_down, up_down_dtod;
  double w_max, w_min, w_max_dtod, w_min_dtod, slope, gamma;
} xb_device_params;

/* proj/include/xbarsim/io.hpp:21-33 plus additive bound management */
typedef struct xb_io_params {
  int32_t dac_bits, adc_bits;
  double input_bound, output_bound, sigma_inp, sigma_out, sigma_w;
  int32_t noise_management, is_perfect;
  int32_t bound_management; /* XB_BM_*; default XB_BM_NONE (= reference) */
  int32_t bm_max_iter;      /* max input halvings under XB_BM_ITERATIVE */
} xb_io_params;

/* proj/include/xbarsim/pulsed.hpp:21-27 */
typedef struct xb_update_params {
  int32_t bl, bl_management, pulse_type;
} xb_update_params;

/* proj/include/xbarsim/tile.hpp:24-36 */
typedef struct xb_temporal_params {
  double decay_rate, decay_dtod, diffusion_sigma, diffusion_dtod, reset_prob, reset_dtod;
} xb_temporal_params;

/* proj/include/xbarsim/tile.hpp:38-44 plus additive MVM precision */
typedef struct xb_tile_config {
  xb_device_params device;
  xb_io_params forward_io, backward_io;
  xb_update_params update;
  int32_t mvm_precision; /* XB_MVM_*; default XB_MVM_TF32X3 (tcgen05 for B >= 16) */
  xb_temporal_params temporal;
  int32_t weight_precision; /* XB_W_*; default XB_W_AUTO */
  int32_t _pad;
} xb_tile_config;

/* Row shard of a larger logical tile: this handle owns global rows
 * [row_begin, row_end) of a d_out_total x d_in tile.  NULL = whole tile.
 * All random draws are keyed on GLOBAL indices, so a P-way sharded tile
 * produces bit-identical results to the unsharded one. */
typedef struct xb_shard {
  int32_t row_begin, row_end, d_out_total, _pad;
} xb_shard;

/* proj/include/xbarsim/inference.hpp:21-36 */
typedef struct xb_inference_model {
  double prog_noise_scale, prog_c0, prog_c1, prog_c2, read_noise_scale;
  double nu_mean, nu_std, t0, nu_min, nu_max;
  int32_t compensation_probes, _pad;
} xb_inference_model;

/* proj/include/xbarsim/compound.hpp:76-91 */
typedef struct xb_transfer_config {
  xb_device_params fast_device, slow_device;
  xb_io_params forward_io, backward_io;
  xb_update_params update;
  int32_t mvm_precision;
  xb_temporal_params temporal;
  int32_t transfer_every, units_in_mbatch;
  double transfer_lr;
  int32_t columns_per_event, has_transfer_io;
  double gamma;
  xb_io_params transfer_io;
} xb_transfer_config;

/* proj/include/xbarsim/compound.hpp:15-28 (vectors -> fixed arrays of
 * n_devices <= XB_MAX_CELL_DEVICES) plus the additive precision mode */
#define XB_MAX_CELL_DEVICES 8
enum { XB_UC_ROUND_ROBIN = 0, XB_UC_ALL_TOGETHER = 1 }; /* UnitCellPolicy order */
typedef struct xb_unitcell_config {
  int32_t n_devices, policy; /* policy default XB_UC_ALL_TOGETHER */
  xb_device_params devices[XB_MAX_CELL_DEVICES];
  double gains[XB_MAX_CELL_DEVICES];
  xb_io_params forward_io, backward_io;
  xb_update_params update;
  int32_t mvm_precision;
  xb_temporal_params temporal;
} xb_unitcell_config;

typedef struct xb_tile xb_tile;
typedef struct xb_transfer xb_transfer;
typedef struct xb_unitcell xb_unitcell;
typedef struct xb_comm xb_comm;

/* ---- library ---- */
int xb_abi_version(void);
const char *xb_last_error(void);
/* 0 when a CUDA device of compute capability 10.x is usable */
int xb_device_check(void);
/* kernel launches issued by this library since load (process-wide) */
uint64_t xb_launch_count(void);
/* measurement helper: device time per launch of n empty kernels issued back
 * to back from C on a fresh stream (best of `reps`), in microseconds -- the
 * launch-latency floor of a step whose work is too small to fill the GPU */
int xb_launch_floor_us(int n, int reps, double *us_per_launch);

/* defaults: the reference's struct initialisers */
void xb_default_device(xb_device_params *p);
void xb_default_io(xb_io_params *p);
void xb_perfect_io(xb_io_params *p); /* proj/src/io.cpp:32-40 */
void xb_default_config(xb_tile_config *c);
void xb_default_transfer_config(xb_transfer_config *c);
void xb_default_inference_model(xb_inference_model *m);
int xb_device_preset(const char *name, xb_device_params *p); /* proj/src/device.cpp:100-132 */

/* ---- AnalogTile ---- */
int xb_tile_create(const xb_tile_config *cfg, int d_out, int d_in, uint64_t seed,
                   const xb_shard *shard, xb_tile **out);
int xb_tile_destroy(xb_tile *t);
int xb_tile_clone(const xb_tile *t, xb_tile **out);
/* local rows, columns, first global row, global rows */
int xb_tile_shape(const xb_tile *t, int *d_out_local, int *d_in, int *row_begin,
                  int *d_out_total);
/* stream used by every call on this handle (cudaStream_t); NULL = own stream */
int xb_tile_set_stream(xb_tile *t, void *stream);
void *xb_tile_stream(const xb_tile *t);

/* weights: local rows x d_in, row-major host fp32; set clips to the per-cell
 * realized bounds (proj/src/tile.cpp:103-119) */
int xb_tile_set_weights(xb_tile *t, const float *w);
int xb_tile_get_weights(const xb_tile *t, float *w);
/* per-cell realization {dw_min_up, dw_min_down, w_max, w_min}, local rows x d_in */
int xb_tile_set_device(xb_tile *t, const float *dw_up, const float *dw_down, const float *w_max,
                       const float *w_min);
int xb_tile_get_device(const xb_tile *t, float *dw_up, float *dw_down, float *w_max,
                       float *w_min);

/* noisy MVM, B samples, host buffers: X [B][d_in] -> Y [B][d_out_local] */
int xb_tile_forward(xb_tile *t, const float *X, int B, float *Y);
int xb_tile_forward_io(xb_tile *t, const float *X, int B, float *Y, const xb_io_params *io);
int xb_tile_forward_noisy(xb_tile *t, const float *X, int B, float *Y, double extra_sigma);
/* D [B][d_out] -> G [B][d_in] (unsharded tiles; see *_partial for shards) */
int xb_tile_backward(xb_tile *t, const float *D, int B, float *G);
/* B sequential pulsed updates; lr[B] per sample (NULL = learning_rate) */
int xb_tile_update(xb_tile *t, const float *X, const float *D, int B, const double *lr);
/* packed pulse trains: xw [B][d_in], dw [B][d_out_local]; bits 0..bl-1 are
 * the slots, bit 31 the sign (1 = negative); flip inverts every pulse */
int xb_tile_apply_trains(xb_tile *t, const uint32_t *xw, const uint32_t *dw, int B, int flip);
/* the trains the NEXT xb_tile_update on these inputs would draw (does not
 * change the tile); bl[B] receives the per-sample train length */
int xb_tile_generate_trains(xb_tile *t, const float *X, const float *D, int B, const double *lr,
                            uint32_t *xw, uint32_t *dw, int32_t *bl);
int xb_tile_temporal_step(xb_tile *t, const xb_temporal_params *tp);
int xb_tile_end_minibatch(xb_tile *t);
int xb_tile_set_learning_rate(xb_tile *t, double lr);
double xb_tile_learning_rate(const xb_tile *t);

/* ---- device-pointer (asynchronous) entries, for callers that keep data in
 *      HBM.  io == NULL selects the tile's forward/backward io. ---- */
int xb_tile_forward_dev(xb_tile *t, const float *dX, int B, float *dY, const xb_io_params *io,
                        double extra_sigma);
int xb_tile_backward_dev(xb_tile *t, const float *dD, int B, float *dG);
/* lr: host array of B learning rates (NULL -> learning_rate for all).
 * dAmaxD: optional device array [B] of the GLOBAL max|d| per sample (row
 * shards: the allreduce-max of xb_rows_amax_dev over ranks); NULL = local. */
int xb_tile_update_dev(xb_tile *t, const float *dX, const float *dD, int B, const double *lr,
                       const float *dAmaxD);
/* backward of a row shard, split around the reduction over ranks:
 *   partial: dP[B][d_in] = sum over local rows of W^T d~ (+ weight-noise fold);
 *            dAmaxD = GLOBAL max|d| per sample (NULL = local)
 *   finish : dG = alpha * ADC(sum_ranks dP + sigma_out xi)
 * Several partials may be in flight before their finishes (a batch split in
 * sample chunks, each chunk's reduction overlapping the next chunk's
 * contraction): finishes must then come in the order of their partials, and
 * the noise draws equal those of one call over the whole batch. */
int xb_tile_backward_partial_dev(xb_tile *t, const float *dD, int B, const float *dAmaxD,
                                 float *dP);
int xb_tile_backward_finish_dev(xb_tile *t, const float *dPsum, int B, const float *dAmaxD,
                                float *dG);
/* out[b] = max_j |V[b][j]| over n entries per row */
int xb_rows_amax_dev(const float *dV, int B, int n, float *dOut, void *stream);
/* block until all work queued on the tile's stream is done */
int xb_tile_synchronize(xb_tile *t);

/* in-stream CUDA-event timing of the kernel phases (for roofline reporting):
 * when enabled, events are recorded on the tile's stream around each phase;
 * xb_tile_read_timing synchronises, returns the summed milliseconds and the
 * launch counts per phase since the last read, and resets them. */
enum { XB_TIMER_PULSE = 0, XB_TIMER_TRAINS = 1, XB_TIMER_FORWARD = 2, XB_TIMER_BACKWARD = 3,
       XB_TIMER_COUNT = 4 };
int xb_tile_set_timing(xb_tile *t, int enable);
int xb_tile_read_timing(xb_tile *t, double *ms, int *counts);

/* ---- row sharding over several GPUs (no reference symbol:
 *      the reference tile is single-device) ----
 * A logical d_out x d_in tile is split by rows over P ranks; rank r creates
 * its handle with an xb_shard and attaches the group's communicator.  The
 * sharded handle then runs the whole-tile semantics of every entry above on
 * its own rows, with the cross-rank reductions enqueued on its stream:
 *   update   -- all-reduce(max) of max|d| before translate (pulsed.cpp:34-51);
 *   forward  -- all-reduce(max) of the bound-management saturation flags
 *               before each re-issue (outputs stay row-sharded: Y[B][local]);
 *   backward -- D is the rank's rows [B][local], G is the full [B][d_in] on
 *               every rank: all-reduce(max) of max|d|, all-reduce(sum) of the
 *               column sums in sample chunks (the reduction of a chunk
 *               overlaps the next chunk's contraction), then noise/ADC/alpha
 *               on the reduced sums (io.cpp:143-146).
 * Random draws are keyed on global rows, so update and forward are bit for
 * bit those of the unsharded tile; the backward differs only by the fp32
 * order of the cross-rank sum.
 * NCCL (over NVLink / NVSwitch) is loaded at run time (XB_NCCL_LIB, else
 * libnccl.so.2). */
#define XB_COMM_ID_BYTES 128
/* ncclGetUniqueId: rank 0 creates it and sends it to the others out of band */
int xb_comm_unique_id(uint8_t *id /* [XB_COMM_ID_BYTES] */);
/* ncclCommInitRank on the current CUDA device (collective over the ranks) */
int xb_comm_create(const uint8_t *id, int nranks, int rank, xb_comm **out);
/* an in-process group of nranks handles out[0..nranks), each to be driven by
 * its own host thread (loopback: several shards may share one device) */
int xb_comm_create_local(int nranks, xb_comm **out);
int xb_comm_destroy(xb_comm *c);
int xb_comm_size(const xb_comm *c);
int xb_comm_rank(const xb_comm *c);
/* route the tile's cross-shard reductions through c (borrowed; NULL detaches) */
int xb_tile_attach_comm(xb_tile *t, xb_comm *c);

/* ---- PCM inference (proj/src/inference.cpp:34-110) ---- */
/* program target (host, local rows x d_in); stores w0 and nu on the device */
int xb_tile_program(xb_tile *t, const float *target, const xb_inference_model *m,
                    uint64_t seed);
int xb_tile_drift_to(xb_tile *t, double time_s);
/* mean over probes of sum_i |forward_noisy(ones)_i| */
int xb_tile_probe_readout(xb_tile *t, const xb_inference_model *m, double *out);
int xb_tile_drift_compensation_factor(xb_tile *t, double baseline, const xb_inference_model *m,
                                      double *alpha);

/* ---- TransferTile / Tiki-Taka (proj/src/compound.cpp:176-293) ---- */
int xb_transfer_create(const xb_transfer_config *cfg, int d_out, int d_in, uint64_t seed,
                       xb_transfer **out);
int xb_transfer_destroy(xb_transfer *t);
int xb_transfer_forward(xb_transfer *t, const float *X, int B, float *Y);
/* forward with sigma_w <- hypot(sigma_w, extra) on both members (compound.cpp:228-238) */
int xb_transfer_forward_noisy(xb_transfer *t, const float *X, int B, float *Y,
                              double extra_sigma);
/* deep copy: both members with their RNG positions, counter and column cursor
   (compound.hpp:109-111) */
int xb_transfer_clone(const xb_transfer *t, xb_transfer **out);
int xb_transfer_backward(xb_transfer *t, const float *D, int B, float *G);
int xb_transfer_update(xb_transfer *t, const float *X, const float *D, int B, const double *lr);
int xb_transfer_end_minibatch(xb_transfer *t);
int xb_transfer_step(xb_transfer *t);
int xb_transfer_get_weights(const xb_transfer *t, float *w);
int xb_transfer_set_weights(xb_transfer *t, const float *w);
long xb_transfer_events(const xb_transfer *t);
xb_tile *xb_transfer_fast(xb_transfer *t);
xb_tile *xb_transfer_slow(xb_transfer *t);

/* ---- UnitCellTile (proj/src/compound.cpp:12-174) ----
 * Members are full B200 tiles (member 0 shares the compound's seed, member k
 * gets derive(seed, "cell_member", k)); the effective weight sum_k g_k W_k is
 * kept in HBM and refreshed after any member changes.  update() draws ONE set
 * of trains per sample from the compound's "update" stream with grain
 * |g| dw_min (round_robin: the member's; all_together: the sum) and fires it on
 * the member(s), flipped for negative gains.  Member handles are borrowed and
 * read-only through the compound. */
void xb_default_unitcell_config(xb_unitcell_config *c);
int xb_unitcell_create(const xb_unitcell_config *cfg, int d_out, int d_in, uint64_t seed,
                       xb_unitcell **out);
int xb_unitcell_destroy(xb_unitcell *u);
int xb_unitcell_clone(const xb_unitcell *u, xb_unitcell **out);
int xb_unitcell_forward(xb_unitcell *u, const float *X, int B, float *Y);
int xb_unitcell_forward_noisy(xb_unitcell *u, const float *X, int B, float *Y,
                              double extra_sigma);
int xb_unitcell_backward(xb_unitcell *u, const float *D, int B, float *G);
/* B sequential UnitCellTile::update calls; lr may be NULL (0.01 each) */
int xb_unitcell_update(xb_unitcell *u, const float *X, const float *D, int B, const double *lr);
int xb_unitcell_get_weights(xb_unitcell *u, float *w);
int xb_unitcell_set_weights(xb_unitcell *u, const float *w);
int xb_unitcell_end_minibatch(xb_unitcell *u);
int xb_unitcell_n_members(const xb_unitcell *u);
xb_tile *xb_unitcell_member(xb_unitcell *u, int k);

#ifdef __cplusplus
}
#endif
#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#endif /* XBTILE_H */
