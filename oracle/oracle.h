/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * C API of the CPU results oracle for the analog-tile hot path. Two
 * implementations share this header:
 *
 *   oracle/xbarsim_oracle.c  plain-C restatement of the reference algorithm
 *                            (liboracle.so, always buildable, travels to the
 *                            GPU box);
 *   oracle/ref_shim.cpp      thin extern "C" wrapper around the reference's
 *                            own sources compiled from /root/reference
 *                            (oracle/_ref/libxbref.so, built only where the
 *                            reference exists, used to pin the restatement).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load either library. The product path
 * (paper_2104_02184_b200/) never links or calls anything here.
 *
 * Every function returns 0 on success and -1 on error (the reference's
 * xbarsim::Error); or_last_error() then holds the message.
 */
#ifndef XB_ORACLE_H
#define XB_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* proj/include/xbarsim/device.hpp:17 (DeviceKind order) */
enum { OR_CONSTANT_STEP = 0, OR_LINEAR_STEP = 1, OR_SOFT_BOUNDS = 2, OR_EXP_STEP = 3 };
/* proj/include/xbarsim/io.hpp:17 */
enum { OR_NM_NONE = 0, OR_NM_ABS_MAX = 1 };
/* proj/include/xbarsim/pulsed.hpp:19 */
enum { OR_PULSE_STOCHASTIC = 0, OR_PULSE_DETERMINISTIC = 1 };

/* proj/include/xbarsim/device.hpp:24-39 */
typedef struct or_device_params {
  int32_t kind;
  int32_t _pad;
  double dw_min, dw_min_dtod, dw_min_std, up_down, up_down_dtod;
  double w_max, w_min, w_max_dtod, w_min_dtod, slope, gamma;
} or_device_params;

/* proj/include/xbarsim/io.hpp:21-33 */
typedef struct or_io_params {
  int32_t dac_bits, adc_bits;
  double input_bound, output_bound, sigma_inp, sigma_out, sigma_w;
  int32_t noise_management, is_perfect;
} or_io_params;

/* proj/include/xbarsim/pulsed.hpp:21-27 */
typedef struct or_update_params {
  int32_t bl, bl_management, pulse_type;
} or_update_params;

/* proj/include/xbarsim/tile.hpp:24-36 */
typedef struct or_temporal_params {
  double decay_rate, decay_dtod, diffusion_sigma, diffusion_dtod, reset_prob, reset_dtod;
} or_temporal_params;

/* proj/include/xbarsim/tile.hpp:38-44 */
typedef struct or_tile_settings {
  or_device_params device;
  or_io_params forward_io, backward_io;
  or_update_params update;
  int32_t _pad;
  or_temporal_params temporal;
} or_tile_settings;

/* proj/include/xbarsim/compound.hpp:76-91 */
typedef struct or_transfer_settings {
  or_device_params fast_device, slow_device;
  or_io_params forward_io, backward_io;
  or_update_params update;
  int32_t _pad;
  or_temporal_params temporal;
  int32_t transfer_every, units_in_mbatch;
  double transfer_lr;
  int32_t columns_per_event, has_transfer_io;
  double gamma;
  or_io_params transfer_io;
} or_transfer_settings;

/* proj/include/xbarsim/inference.hpp:21-36 */
typedef struct or_inference_model {
  double prog_noise_scale, prog_c0, prog_c1, prog_c2, read_noise_scale;
  double nu_mean, nu_std, t0, nu_min, nu_max;
  int32_t compensation_probes, _pad;
} or_inference_model;

/* proj/include/xbarsim/compound.hpp:15-28 (vectors -> fixed arrays) */
#define OR_MAX_CELL_DEVICES 8
enum { OR_UC_ROUND_ROBIN = 0, OR_UC_ALL_TOGETHER = 1 };
typedef struct or_unitcell_settings {
  int32_t n_devices, policy;
  or_device_params devices[OR_MAX_CELL_DEVICES];
  double gains[OR_MAX_CELL_DEVICES];
  or_io_params forward_io, backward_io;
  or_update_params update;
  int32_t _pad;
  or_temporal_params temporal;
} or_unitcell_settings;

typedef struct or_rng or_rng;
typedef struct or_tile or_tile;
typedef struct or_transfer or_transfer;
typedef struct or_unitcell or_unitcell;

const char *or_last_error(void);
/* "restatement" or "reference" -- which implementation this library is */
const char *or_impl_name(void);

/* defaults, exactly the reference's struct initialisers / presets */
void or_default_device(or_device_params *p);
void or_default_io(or_io_params *p);
void or_perfect_io(or_io_params *p);
void or_default_update(or_update_params *p);
void or_default_temporal(or_temporal_params *p);
void or_default_tile_settings(or_tile_settings *s);
void or_default_transfer_settings(or_transfer_settings *s);
void or_default_inference_model(or_inference_model *m);
int or_device_preset(const char *name, or_device_params *p);

/* ---- RngStream (proj/src/rng.cpp) ---- */
or_rng *or_rng_new(uint64_t seed);
or_rng *or_rng_derive(const or_rng *r, const char *name);
or_rng *or_rng_derive_idx(const or_rng *r, const char *name, uint64_t index);
void or_rng_free(or_rng *r);
uint64_t or_rng_base_seed(const or_rng *r);
uint64_t or_rng_next_u64(or_rng *r);
double or_rng_uniform(or_rng *r);
double or_rng_gauss(or_rng *r);
int or_rng_bernoulli(or_rng *r, double p);

/* ---- converters / MVM (proj/src/io.cpp) ---- */
double or_quantize_uniform(double v, double bound, int bits);
void or_with_extra_weight_noise(const or_io_params *io, double extra, or_io_params *out);
/* W row-major rows x cols; out has cols (transposed) or rows entries */
int or_analog_matvec(const double *w, int rows, int cols, const double *in,
                     const or_io_params *io, or_rng *rng, int transposed, double *out);

/* ---- devices (proj/src/device.cpp) ---- */
/* cell[6] = {dw_min_up, dw_min_down, w_max, w_min, slope, gamma} */
int or_realize_cell(const or_device_params *p, or_rng *rng, double *cell);
double or_apply_pulse(const double *cell, double w, int up, int kind, double dw_min_std,
                      or_rng *rng);

/* ---- pulsed update (proj/src/pulsed.cpp) ---- */
int or_translate(const double *x, int nx, const double *d, int nd, double lr, double dw_min,
                 const or_update_params *up, int *bl, double *px, double *pd, int *sx, int *sd);
/* bits slot-major: xbits[t*nx + j], dbits[t*nd + i] */
int or_generate_trains(int bl, const double *px, int nx, const double *pd, int nd, or_rng *rng,
                       uint8_t *xbits, uint8_t *dbits);

/* ---- AnalogTile (proj/src/tile.cpp) ---- */
or_tile *or_tile_new(int d_out, int d_in, const or_tile_settings *s, uint64_t seed);
or_tile *or_tile_clone(const or_tile *t);
void or_tile_free(or_tile *t);
int or_tile_forward(or_tile *t, const double *x, double *y);
int or_tile_backward(or_tile *t, const double *d, double *g);
int or_tile_update(or_tile *t, const double *x, const double *d, double lr);
int or_tile_forward_noisy(or_tile *t, const double *x, double extra_sigma, double *y);
int or_tile_forward_with_io(or_tile *t, const double *x, const or_io_params *io, double *y);
int or_tile_get_weights(const or_tile *t, double *w);
int or_tile_set_weights(or_tile *t, const double *w);
/* per-cell realization, row-major arrays of d_out*d_in */
int or_tile_get_device(const or_tile *t, double *dw_up, double *dw_down, double *w_max,
                       double *w_min);
int or_tile_apply_pulse_trains(or_tile *t, int bl, const uint8_t *xbits, const uint8_t *dbits,
                               const int *sign_x, const int *sign_d, int flip);
int or_tile_apply_temporal_step(or_tile *t, const or_temporal_params *tp);
int or_tile_end_minibatch(or_tile *t);

/* ---- TransferTile (proj/src/compound.cpp:176-293) ---- */
or_transfer *or_transfer_new(int d_out, int d_in, const or_transfer_settings *s, uint64_t seed);
void or_transfer_free(or_transfer *t);
int or_transfer_forward(or_transfer *t, const double *x, double *y);
int or_transfer_backward(or_transfer *t, const double *d, double *g);
int or_transfer_update(or_transfer *t, const double *x, const double *d, double lr);
int or_transfer_end_minibatch(or_transfer *t);
int or_transfer_step(or_transfer *t);
int or_transfer_get_weights(const or_transfer *t, double *w);
int or_transfer_set_weights(or_transfer *t, const double *w);
long or_transfer_events(const or_transfer *t);
/* borrowed handles to the member tiles (valid while t lives) */
or_tile *or_transfer_fast(or_transfer *t);
or_tile *or_transfer_slow(or_transfer *t);


/* UnitCellTile -- proj/src/compound.cpp:12-174 */
void or_default_unitcell_settings(or_unitcell_settings *s);
or_unitcell *or_unitcell_new(int d_out, int d_in, const or_unitcell_settings *s, uint64_t seed);
or_unitcell *or_unitcell_clone(const or_unitcell *t);
void or_unitcell_free(or_unitcell *t);
int or_unitcell_forward(or_unitcell *t, const double *x, double *y);
int or_unitcell_backward(or_unitcell *t, const double *d, double *g);
int or_unitcell_forward_noisy(or_unitcell *t, const double *x, double extra_sigma, double *y);
int or_unitcell_update(or_unitcell *t, const double *x, const double *d, double lr);
int or_unitcell_get_weights(const or_unitcell *t, double *w);
int or_unitcell_set_weights(or_unitcell *t, const double *w);
int or_unitcell_end_minibatch(or_unitcell *t);
int or_unitcell_n_members(const or_unitcell *t);
or_tile *or_unitcell_member(or_unitcell *t, int k);
/* ---- PCM inference (proj/src/inference.cpp:14-110) ---- */
int or_program(or_tile *t, const double *target, const or_inference_model *m, or_rng *rng,
               double *w0_out, double *nu_out);
int or_drift_to(or_tile *t, const double *w0, const double *nu, double t0, double time_s);
int or_probe_readout(or_tile *t, const or_inference_model *m, double *out);
int or_drift_compensation_factor(or_tile *t, double baseline, const or_inference_model *m,
                                 double *alpha);

#ifdef __cplusplus
}
#endif
#endif
