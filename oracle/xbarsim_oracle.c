/*
 * xbarsim_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker).
 *
 * A plain-C restatement of the reference analog-tile hot path
 * (xbarsim, /root/reference/proj), double precision, single threaded, with
 * the reference's own random-number scheme (std::mt19937_64 seeded through
 * splitmix64 / FNV-1a stream derivation, 53-bit uniforms, Box-Muller with a
 * spare).  Every function cites the reference file:line it restates.  Given
 * the same inputs and seeds it reproduces the reference bit for bit (same
 * operation order, same libm calls); tests/test_oracle_pin.py checks that
 * against oracle/_ref (the reference compiled from its own sources) and
 * tests/golden/ fixtures generated from it.
 *
 * Parity pinned: yes -- against oracle/_ref and the tests/golden fixtures.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline /
 * --impl reference) may load this library.  The CUDA product path never
 * does.
 */
#include "oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

static int fail(const char *msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return -1;
}

const char *or_last_error(void) { return g_err; }
const char *or_impl_name(void) { return "restatement"; }

/* std::max / std::min / std::clamp exactly as libstdc++ defines them */
static inline double smax(double a, double b) { return (a < b) ? b : a; }
static inline double smin(double a, double b) { return (b < a) ? b : a; }
static inline double sclamp(double v, double lo, double hi) {
  return (v < lo) ? lo : ((hi < v) ? hi : v);
}

/* ======================================================================
 * RngStream -- proj/src/rng.cpp:14-71, proj/include/xbarsim/rng.hpp:18-39
 * ====================================================================== */

#define MT_N 312
#define MT_M 156

struct or_rng {
  uint64_t seed;
  uint64_t mt[MT_N];
  int mti;
  int has_spare;
  double spare;
};

/* proj/src/rng.cpp:14-21 */
static uint64_t fnv1a(const char *s) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (; *s; ++s) {
    h ^= (unsigned char)*s;
    h *= 0x100000001b3ull;
  }
  return h;
}

/* proj/src/rng.cpp:24-29 (splitmix64 finaliser) */
static uint64_t mix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

/* std::mt19937_64(seed) -- the standard (C++11 [rand.eng.mers]) engine */
static void mt_seed(or_rng *r, uint64_t s) {
  r->mt[0] = s;
  for (int i = 1; i < MT_N; ++i) {
    r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  }
  r->mti = MT_N;
}

static uint64_t mt_next(or_rng *r) {
  static const uint64_t mag[2] = {0ull, 0xB5026F5AA96619E9ull};
  const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
  if (r->mti >= MT_N) {
    int i;
    for (i = 0; i < MT_N - MT_M; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + MT_M] ^ (x >> 1) ^ mag[x & 1ull];
    }
    for (; i < MT_N - 1; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + (MT_M - MT_N)] ^ (x >> 1) ^ mag[x & 1ull];
    }
    uint64_t x = (r->mt[MT_N - 1] & UM) | (r->mt[0] & LM);
    r->mt[MT_N - 1] = r->mt[MT_M - 1] ^ (x >> 1) ^ mag[x & 1ull];
    r->mti = 0;
  }
  uint64_t x = r->mt[r->mti++];
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71D67FFFEDA60000ull;
  x ^= (x << 37) & 0xFFF7EEE000000000ull;
  x ^= (x >> 43);
  return x;
}

/* proj/src/rng.cpp:33 -- RngStream(seed): seed_(seed), gen_(mix(seed)) */
static void rng_init(or_rng *r, uint64_t seed) {
  r->seed = seed;
  mt_seed(r, mix(seed));
  r->has_spare = 0;
  r->spare = 0.0;
}

or_rng *or_rng_new(uint64_t seed) {
  or_rng *r = (or_rng *)malloc(sizeof(or_rng));
  rng_init(r, seed);
  return r;
}

/* proj/src/rng.cpp:35-37 */
static uint64_t derive_seed(uint64_t base, const char *name) { return mix(base ^ fnv1a(name)); }
/* proj/src/rng.cpp:39-41 */
static uint64_t derive_seed_idx(uint64_t base, const char *name, uint64_t idx) {
  return mix(mix(base ^ fnv1a(name)) + idx);
}

or_rng *or_rng_derive(const or_rng *r, const char *name) {
  return or_rng_new(derive_seed(r->seed, name));
}
or_rng *or_rng_derive_idx(const or_rng *r, const char *name, uint64_t index) {
  return or_rng_new(derive_seed_idx(r->seed, name, index));
}
void or_rng_free(or_rng *r) { free(r); }
uint64_t or_rng_base_seed(const or_rng *r) { return r->seed; }
uint64_t or_rng_next_u64(or_rng *r) { return mt_next(r); }

/* proj/src/rng.cpp:45-47 */
double or_rng_uniform(or_rng *r) { return (double)(mt_next(r) >> 11) * 0x1.0p-53; }

/* proj/src/rng.cpp:49-61 */
double or_rng_gauss(or_rng *r) {
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  double u1 = 1.0 - or_rng_uniform(r);
  double u2 = or_rng_uniform(r);
  double rad = sqrt(-2.0 * log(u1));
  double a = 2.0 * M_PI * u2;
  r->spare = rad * sin(a);
  r->has_spare = 1;
  return rad * cos(a);
}

/* proj/src/rng.cpp:63-71 */
int or_rng_bernoulli(or_rng *r, double p) {
  if (p <= 0.0) return 0;
  if (p >= 1.0) return 1;
  return or_rng_uniform(r) < p;
}

/* ======================================================================
 * Defaults -- struct initialisers of the reference headers
 * ====================================================================== */

/* proj/include/xbarsim/device.hpp:24-39 */
void or_default_device(or_device_params *p) {
  memset(p, 0, sizeof *p);
  p->kind = OR_CONSTANT_STEP;
  p->dw_min = 0.001;
  p->w_max = 1.0;
  p->w_min = -1.0;
  p->slope = 1.0;
  p->gamma = 2.0;
}

/* proj/include/xbarsim/io.hpp:21-33 */
void or_default_io(or_io_params *p) {
  memset(p, 0, sizeof *p);
  p->dac_bits = 7;
  p->adc_bits = 9;
  p->input_bound = 1.0;
  p->output_bound = 12.0;
  p->sigma_out = 0.06;
  p->noise_management = OR_NM_ABS_MAX;
}

/* proj/src/io.cpp:32-40 */
void or_perfect_io(or_io_params *p) {
  or_default_io(p);
  p->is_perfect = 1;
  p->dac_bits = 0;
  p->adc_bits = 0;
  p->sigma_out = 0.0;
  p->noise_management = OR_NM_NONE;
}

/* proj/include/xbarsim/pulsed.hpp:21-27 */
void or_default_update(or_update_params *p) {
  p->bl = 31;
  p->bl_management = 0;
  p->pulse_type = OR_PULSE_STOCHASTIC;
}

void or_default_temporal(or_temporal_params *p) { memset(p, 0, sizeof *p); }

void or_default_tile_settings(or_tile_settings *s) {
  memset(s, 0, sizeof *s);
  or_default_device(&s->device);
  or_default_io(&s->forward_io);
  or_default_io(&s->backward_io);
  or_default_update(&s->update);
  or_default_temporal(&s->temporal);
}

/* proj/include/xbarsim/compound.hpp:76-91 */
void or_default_transfer_settings(or_transfer_settings *s) {
  memset(s, 0, sizeof *s);
  or_default_device(&s->fast_device);
  or_default_device(&s->slow_device);
  or_default_io(&s->forward_io);
  or_default_io(&s->backward_io);
  or_default_update(&s->update);
  or_default_temporal(&s->temporal);
  s->transfer_every = 1;
  s->units_in_mbatch = 0;
  s->transfer_lr = 0.1;
  s->columns_per_event = 1;
  s->gamma = 0.0;
  s->has_transfer_io = 0;
  or_default_io(&s->transfer_io);
}

/* proj/include/xbarsim/inference.hpp:21-36 */
void or_default_inference_model(or_inference_model *m) {
  memset(m, 0, sizeof *m);
  m->prog_noise_scale = 1.0;
  m->prog_c0 = 0.26;
  m->prog_c1 = 1.66;
  m->prog_c2 = 0.33;
  m->read_noise_scale = 0.0;
  m->nu_mean = 0.06;
  m->nu_std = 0.03;
  m->t0 = 20.0;
  m->nu_min = 0.0;
  m->nu_max = 1.0;
  m->compensation_probes = 10;
}

/* proj/src/device.cpp:100-132 */
int or_device_preset(const char *name, or_device_params *p) {
  or_default_device(p);
  if (strcmp(name, "ideal") == 0) {
    p->kind = OR_CONSTANT_STEP;
    p->dw_min = 1e-6;
    p->w_max = 1.0;
    p->w_min = -1.0;
    return 0;
  }
  if (strcmp(name, "reram_sb") == 0) {
    p->kind = OR_SOFT_BOUNDS;
    p->dw_min = 0.002;
    p->dw_min_dtod = 0.3;
    p->dw_min_std = 0.3;
    p->w_max = 0.6;
    p->w_min = -0.6;
    p->up_down_dtod = 0.01;
    return 0;
  }
  if (strcmp(name, "reram_es") == 0) {
    p->kind = OR_EXP_STEP;
    p->dw_min = 0.001;
    p->dw_min_dtod = 0.3;
    p->dw_min_std = 0.3;
    p->w_max = 0.6;
    p->w_min = -0.6;
    p->up_down = 0.1;
    p->up_down_dtod = 0.01;
    p->gamma = 2.0;
    return 0;
  }
  char buf[256];
  snprintf(buf, sizeof buf, "device preset: unknown name '%s'", name);
  return fail(buf);
}

/* ======================================================================
 * Validation -- error messages name the field like the reference
 * ====================================================================== */

/* proj/src/io.cpp:14-30 */
static int io_validate(const or_io_params *io, const char *ctx) {
  char buf[256];
  if (io->dac_bits < 0) {
    snprintf(buf, sizeof buf, "%s.dac_bits: must be >= 0", ctx);
    return fail(buf);
  }
  if (io->adc_bits < 0) {
    snprintf(buf, sizeof buf, "%s.adc_bits: must be >= 0", ctx);
    return fail(buf);
  }
  if (!(io->input_bound > 0.0)) {
    snprintf(buf, sizeof buf, "%s.input_bound: must be > 0", ctx);
    return fail(buf);
  }
  if (!(io->output_bound > 0.0)) {
    snprintf(buf, sizeof buf, "%s.output_bound: must be > 0", ctx);
    return fail(buf);
  }
  if (io->sigma_inp < 0.0 || io->sigma_out < 0.0 || io->sigma_w < 0.0) {
    snprintf(buf, sizeof buf, "%s: noise sigmas must be >= 0", ctx);
    return fail(buf);
  }
  return 0;
}

/* proj/src/device.cpp:13-24 */
static int device_validate(const or_device_params *p, const char *ctx) {
  char buf[256];
  if (!(p->dw_min > 0.0)) {
    snprintf(buf, sizeof buf, "%s.dw_min: must be > 0", ctx);
    return fail(buf);
  }
  if (!(p->w_min < 0.0 && 0.0 < p->w_max)) {
    snprintf(buf, sizeof buf, "%s: requires w_min < 0 < w_max", ctx);
    return fail(buf);
  }
  if (p->dw_min_dtod < 0.0 || p->dw_min_std < 0.0 || p->up_down_dtod < 0.0 ||
      p->w_max_dtod < 0.0 || p->w_min_dtod < 0.0) {
    snprintf(buf, sizeof buf, "%s: dtod/std spreads must be >= 0", ctx);
    return fail(buf);
  }
  return 0;
}

/* proj/src/pulsed.cpp:13-17 */
static int update_validate(const or_update_params *u, const char *ctx) {
  char buf[256];
  if (u->bl < 1) {
    snprintf(buf, sizeof buf, "%s.bl: must be >= 1", ctx);
    return fail(buf);
  }
  return 0;
}

/* proj/src/tile.cpp:13-23 */
static int temporal_validate(const or_temporal_params *tp, const char *ctx) {
  char buf[256];
  if (tp->decay_rate < 0.0 || tp->diffusion_sigma < 0.0) {
    snprintf(buf, sizeof buf, "%s: decay_rate and diffusion_sigma must be >= 0", ctx);
    return fail(buf);
  }
  if (tp->reset_prob < 0.0 || tp->reset_prob > 1.0) {
    snprintf(buf, sizeof buf, "%s.reset_prob: must be in [0, 1]", ctx);
    return fail(buf);
  }
  if (tp->decay_dtod < 0.0 || tp->diffusion_dtod < 0.0 || tp->reset_dtod < 0.0) {
    snprintf(buf, sizeof buf, "%s: dtod spreads must be >= 0", ctx);
    return fail(buf);
  }
  return 0;
}

/* ======================================================================
 * Converters and the noisy MVM -- proj/src/io.cpp:42-149
 * ====================================================================== */

/* proj/src/io.cpp:42-56 */
double or_quantize_uniform(double v, double bound, int bits) {
  if (v == 0.0) return 0.0;
  v = sclamp(v, -bound, bound);
  if (bits <= 0) return v;
  const double levels = exp2((double)bits);
  const double step = 2.0 * bound / levels;
  double k = round((v + bound - 0.5 * step) / step);
  k = sclamp(k, 0.0, levels - 1.0);
  return -bound + (k + 0.5) * step;
}

/* proj/src/io.cpp:74-91 */
void or_with_extra_weight_noise(const or_io_params *io, double extra, or_io_params *out) {
  *out = *io;
  if (extra <= 0.0) return;
  if (out->is_perfect) {
    or_default_io(out);
    out->dac_bits = 0;
    out->adc_bits = 0;
    out->input_bound = INFINITY;
    out->output_bound = INFINITY;
    out->sigma_out = 0.0;
    out->noise_management = OR_NM_NONE;
  }
  out->is_perfect = 0;
  out->sigma_w = hypot(out->sigma_w, extra);
}

/* proj/include/xbarsim/matrix.hpp:74-80 */
static double max_abs(const double *v, int n) {
  double m = 0.0;
  for (int i = 0; i < n; ++i) m = smax(m, fabs(v[i]));
  return m;
}

/* proj/src/io.cpp:93-149 (and matrix.hpp:52-72 for the perfect path) */
int or_analog_matvec(const double *w, int rows, int cols, const double *in,
                     const or_io_params *io, or_rng *rng, int transposed, double *out) {
  const int in_size = transposed ? rows : cols;
  const int out_size = transposed ? cols : rows;

  if (io->is_perfect) {
    if (!transposed) {
      /* matrix.hpp:52-62 */
      for (int i = 0; i < rows; ++i) {
        double acc = 0.0;
        for (int j = 0; j < cols; ++j) acc += w[(size_t)i * cols + j] * in[j];
        out[i] = acc;
      }
    } else {
      /* matrix.hpp:64-72: row-outer accumulation order */
      for (int j = 0; j < cols; ++j) out[j] = 0.0;
      for (int i = 0; i < rows; ++i)
        for (int j = 0; j < cols; ++j) out[j] += w[(size_t)i * cols + j] * in[i];
    }
    return 0;
  }

  /* io.cpp:107-115 zero input: output noise only */
  if (max_abs(in, in_size) == 0.0) {
    for (int i = 0; i < out_size; ++i) out[i] = 0.0;
    if (io->sigma_out > 0.0) {
      for (int i = 0; i < out_size; ++i)
        out[i] = or_quantize_uniform(io->sigma_out * or_rng_gauss(rng), io->output_bound,
                                     io->adc_bits);
    }
    return 0;
  }

  double alpha = 1.0;
  if (io->noise_management == OR_NM_ABS_MAX) alpha = max_abs(in, in_size);

  double *x = (double *)malloc(sizeof(double) * (size_t)in_size);
  for (int j = 0; j < in_size; ++j) {
    double v = or_quantize_uniform(in[j] / alpha, io->input_bound, io->dac_bits);
    if (io->sigma_inp > 0.0) v += io->sigma_inp * or_rng_gauss(rng);
    x[j] = v;
  }
  for (int i = 0; i < out_size; ++i) {
    double acc = 0.0;
    for (int j = 0; j < in_size; ++j) {
      double wv = transposed ? w[(size_t)j * cols + i] : w[(size_t)i * cols + j];
      if (io->sigma_w > 0.0) wv += io->sigma_w * or_rng_gauss(rng);
      acc += wv * x[j];
    }
    if (io->sigma_out > 0.0) acc += io->sigma_out * or_rng_gauss(rng);
    out[i] = alpha * or_quantize_uniform(acc, io->output_bound, io->adc_bits);
  }
  free(x);
  return 0;
}

/* ======================================================================
 * Device models -- proj/src/device.cpp:26-98
 * ====================================================================== */

/* proj/src/device.cpp:26-46 */
int or_realize_cell(const or_device_params *p, or_rng *rng, double *cell) {
  const double xi_dw = or_rng_gauss(rng);
  const double xi_ud = or_rng_gauss(rng);
  const double xi_max = or_rng_gauss(rng);
  const double xi_min = or_rng_gauss(rng);
  const double floor_ = 0.01 * p->dw_min;
  const double dw = smax(p->dw_min * (1.0 + p->dw_min_dtod * xi_dw), floor_);
  const double bias = p->up_down + p->up_down_dtod * xi_ud;
  cell[0] = smax(dw * (1.0 + bias), floor_);
  cell[1] = smax(dw * (1.0 - bias), floor_);
  cell[2] = smax(p->w_max * (1.0 + p->w_max_dtod * xi_max), 0.01 * p->w_max);
  cell[3] = smin(p->w_min * (1.0 + p->w_min_dtod * xi_min), 0.01 * p->w_min);
  cell[4] = p->slope;
  cell[5] = p->gamma;
  return 0;
}

/* proj/src/device.cpp:48-77 */
double or_apply_pulse(const double *cell, double w, int up, int kind, double dw_min_std,
                      or_rng *rng) {
  double step = 0.0;
  switch (kind) {
  case OR_CONSTANT_STEP:
    step = up ? cell[0] : cell[1];
    break;
  case OR_SOFT_BOUNDS:
    step = up ? cell[0] * (1.0 - w / cell[2]) : cell[1] * (1.0 - w / cell[3]);
    break;
  case OR_LINEAR_STEP:
    step = up ? cell[0] * (1.0 - cell[4] * w) : cell[1] * (1.0 + cell[4] * w);
    break;
  case OR_EXP_STEP: {
    const double range = cell[2] - cell[3];
    step = up ? cell[0] * exp(-cell[5] * (w - cell[3]) / range)
              : cell[1] * exp(-cell[5] * (cell[2] - w) / range);
    break;
  }
  }
  if (dw_min_std > 0.0) step *= 1.0 + dw_min_std * or_rng_gauss(rng);
  w += up ? step : -step;
  return sclamp(w, cell[3], cell[2]);
}

/* ======================================================================
 * Pulsed update -- proj/src/pulsed.cpp:25-148
 * ====================================================================== */

static int sign_of(double v) { return (v > 0.0) - (v < 0.0); }

/* proj/src/pulsed.cpp:25-66 */
int or_translate(const double *x, int nx, const double *d, int nd, double lr, double dw_min,
                 const or_update_params *up, int *bl_out, double *px, double *pd, int *sx,
                 int *sd) {
  if (!(lr > 0.0)) return fail("translate: learning rate must be > 0");
  if (!(dw_min > 0.0)) return fail("translate: dw_min must be > 0");
  const double x_amax = max_abs(x, nx);
  const double d_amax = max_abs(d, nd);
  int bl = up->bl;
  if (up->bl_management) {
    const double quanta = lr * x_amax * d_amax / dw_min;
    int c = (int)ceil(up->bl * smin(1.0, quanta));
    bl = c > 1 ? c : 1; /* std::max(1, c) */
  }
  const double amp = sqrt(lr / (dw_min * bl));
  double x_scale = 1.0, d_scale = 1.0;
  if (x_amax > 0.0 && d_amax > 0.0) {
    x_scale = sqrt(d_amax / x_amax);
    d_scale = 1.0 / x_scale;
  }
  for (int j = 0; j < nx; ++j) {
    px[j] = smin(1.0, amp * fabs(x[j]) * x_scale);
    sx[j] = sign_of(x[j]);
  }
  for (int i = 0; i < nd; ++i) {
    pd[i] = smin(1.0, amp * fabs(d[i]) * d_scale);
    sd[i] = sign_of(d[i]);
  }
  *bl_out = bl;
  return 0;
}

/* proj/src/pulsed.cpp:68-88 */
int or_generate_trains(int bl, const double *px, int nx, const double *pd, int nd, or_rng *rng,
                       uint8_t *xbits, uint8_t *dbits) {
  for (int t = 0; t < bl; ++t)
    for (int j = 0; j < nx; ++j) xbits[(size_t)t * nx + j] = or_rng_bernoulli(rng, px[j]) ? 1 : 0;
  for (int t = 0; t < bl; ++t)
    for (int i = 0; i < nd; ++i) dbits[(size_t)t * nd + i] = or_rng_bernoulli(rng, pd[i]) ? 1 : 0;
  return 0;
}

/* ======================================================================
 * AnalogTile -- proj/src/tile.cpp:41-171
 * ====================================================================== */

struct or_tile {
  int d_out, d_in;
  or_tile_settings s;
  double *cells;   /* [d_out*d_in][6] realization, proj/src/device.cpp:79-88 */
  double *w;       /* [d_out*d_in] */
  double lr;
  or_rng rng_forward, rng_backward, rng_update, rng_temporal;
  double *xi_decay, *xi_diffusion, *xi_reset;
};

static double cell_clip(const or_tile *t, size_t c, double w) {
  return sclamp(w, t->cells[c * 6 + 3], t->cells[c * 6 + 2]);
}

/* proj/src/tile.cpp:41-63 */
or_tile *or_tile_new(int d_out, int d_in, const or_tile_settings *s, uint64_t seed) {
  if (d_out < 1 || d_in < 1) {
    fail("tile: dimensions must be >= 1");
    return NULL;
  }
  if (io_validate(&s->forward_io, "forward_io") || io_validate(&s->backward_io, "backward_io") ||
      update_validate(&s->update, "update") || temporal_validate(&s->temporal, "temporal"))
    return NULL;
  if (device_validate(&s->device, "device")) return NULL; /* device.cpp:81 */
  or_tile *t = (or_tile *)calloc(1, sizeof(or_tile));
  t->d_out = d_out;
  t->d_in = d_in;
  t->s = *s;
  t->lr = 0.01;
  or_rng base;
  rng_init(&base, seed);
  rng_init(&t->rng_forward, derive_seed(seed, "forward"));
  rng_init(&t->rng_backward, derive_seed(seed, "backward"));
  rng_init(&t->rng_update, derive_seed(seed, "update"));
  rng_init(&t->rng_temporal, derive_seed(seed, "temporal"));
  const size_t n = (size_t)d_out * d_in;
  t->cells = (double *)malloc(sizeof(double) * 6 * n);
  t->w = (double *)calloc(n, sizeof(double));
  or_rng init;
  rng_init(&init, derive_seed(seed, "realize")); /* tile.cpp:27 */
  for (size_t c = 0; c < n; ++c) or_realize_cell(&t->s.device, &init, t->cells + 6 * c);
  or_rng tinit;
  rng_init(&tinit, derive_seed(seed, "temporal_init")); /* tile.cpp:59-62 */
  t->xi_decay = (double *)malloc(sizeof(double) * n);
  t->xi_diffusion = (double *)malloc(sizeof(double) * n);
  t->xi_reset = (double *)malloc(sizeof(double) * n);
  for (size_t c = 0; c < n; ++c) t->xi_decay[c] = or_rng_gauss(&tinit);
  for (size_t c = 0; c < n; ++c) t->xi_diffusion[c] = or_rng_gauss(&tinit);
  for (size_t c = 0; c < n; ++c) t->xi_reset[c] = or_rng_gauss(&tinit);
  (void)base;
  return t;
}

static double *dup(const double *p, size_t n) {
  double *q = (double *)malloc(sizeof(double) * n);
  memcpy(q, p, sizeof(double) * n);
  return q;
}

/* proj/include/xbarsim/tile.hpp:91 (clone = deep copy) */
or_tile *or_tile_clone(const or_tile *t) {
  or_tile *c = (or_tile *)malloc(sizeof(or_tile));
  *c = *t;
  const size_t n = (size_t)t->d_out * t->d_in;
  c->cells = dup(t->cells, 6 * n);
  c->w = dup(t->w, n);
  c->xi_decay = dup(t->xi_decay, n);
  c->xi_diffusion = dup(t->xi_diffusion, n);
  c->xi_reset = dup(t->xi_reset, n);
  return c;
}

void or_tile_free(or_tile *t) {
  if (!t) return;
  free(t->cells);
  free(t->w);
  free(t->xi_decay);
  free(t->xi_diffusion);
  free(t->xi_reset);
  free(t);
}

/* proj/src/tile.cpp:65-75 */
static int check_input(const double *v, int expected, const char *what) {
  char buf[256];
  (void)expected;
  for (int i = 0; i < expected; ++i) {
    if (!isfinite(v[i])) {
      snprintf(buf, sizeof buf, "%s: non-finite entry", what);
      return fail(buf);
    }
  }
  return 0;
}

/* proj/src/tile.cpp:77-80 */
int or_tile_forward(or_tile *t, const double *x, double *y) {
  if (check_input(x, t->d_in, "forward")) return -1;
  return or_analog_matvec(t->w, t->d_out, t->d_in, x, &t->s.forward_io, &t->rng_forward, 0, y);
}

/* proj/src/tile.cpp:82-85 */
int or_tile_backward(or_tile *t, const double *d, double *g) {
  if (check_input(d, t->d_out, "backward")) return -1;
  return or_analog_matvec(t->w, t->d_out, t->d_in, d, &t->s.backward_io, &t->rng_backward, 1, g);
}

/* proj/src/tile.cpp:87-90 */
int or_tile_forward_with_io(or_tile *t, const double *x, const or_io_params *io, double *y) {
  if (check_input(x, t->d_in, "forward")) return -1;
  return or_analog_matvec(t->w, t->d_out, t->d_in, x, io, &t->rng_forward, 0, y);
}

/* proj/src/tile.cpp:92-95 */
int or_tile_forward_noisy(or_tile *t, const double *x, double extra_sigma, double *y) {
  or_io_params io;
  or_with_extra_weight_noise(&t->s.forward_io, extra_sigma, &io);
  return or_tile_forward_with_io(t, x, &io, y);
}

/* proj/src/pulsed.cpp:90-114 with trains given slot-major */
static void apply_coincidences(or_tile *t, int bl, const uint8_t *xb, const uint8_t *db,
                               const int *sx, const int *sd, int flip) {
  const int nr = t->d_out, nc = t->d_in;
  for (int s = 0; s < bl; ++s) {
    for (int i = 0; i < nr; ++i) {
      if (!db[(size_t)s * nr + i]) continue;
      for (int j = 0; j < nc; ++j) {
        if (!xb[(size_t)s * nc + j]) continue;
        const int sdi = flip ? -sd[i] : sd[i]; /* tile.cpp:164-167 */
        const int sg = sdi * sx[j];
        if (sg == 0) continue;
        const size_t c = (size_t)i * nc + j;
        t->w[c] = or_apply_pulse(t->cells + 6 * c, t->w[c], sg > 0, t->s.device.kind,
                                 t->s.device.dw_min_std, &t->rng_update);
      }
    }
  }
}

/* proj/src/tile.cpp:97-101 -> proj/src/pulsed.cpp:116-148 */
int or_tile_update(or_tile *t, const double *x, const double *d, double lr) {
  if (check_input(x, t->d_in, "update(x)")) return -1;
  if (check_input(d, t->d_out, "update(d)")) return -1;
  const int nr = t->d_out, nc = t->d_in;
  if (lr == 0.0 || max_abs(x, nc) == 0.0 || max_abs(d, nr) == 0.0) return 0; /* :122-124 */
  double *px = (double *)malloc(sizeof(double) * nc);
  double *pd = (double *)malloc(sizeof(double) * nr);
  int *sx = (int *)malloc(sizeof(int) * nc);
  int *sd = (int *)malloc(sizeof(int) * nr);
  int bl;
  int rc = or_translate(x, nc, d, nr, lr, t->s.device.dw_min, &t->s.update, &bl, px, pd, sx, sd);
  if (rc == 0) {
    if (t->s.update.pulse_type == OR_PULSE_DETERMINISTIC) {
      /* pulsed.cpp:128-144 */
      for (int i = 0; i < nr; ++i) {
        for (int j = 0; j < nc; ++j) {
          const int sg = sd[i] * sx[j];
          if (sg == 0) continue;
          const long count = lround(bl * pd[i] * px[j]);
          const size_t c = (size_t)i * nc + j;
          for (long k = 0; k < count; ++k)
            t->w[c] = or_apply_pulse(t->cells + 6 * c, t->w[c], sg > 0, t->s.device.kind,
                                     t->s.device.dw_min_std, &t->rng_update);
        }
      }
    } else {
      uint8_t *xb = (uint8_t *)malloc((size_t)bl * nc);
      uint8_t *db = (uint8_t *)malloc((size_t)bl * nr);
      or_generate_trains(bl, px, nc, pd, nr, &t->rng_update, xb, db);
      apply_coincidences(t, bl, xb, db, sx, sd, 0);
      free(xb);
      free(db);
    }
  }
  free(px);
  free(pd);
  free(sx);
  free(sd);
  return rc;
}

int or_tile_get_weights(const or_tile *t, double *w) {
  memcpy(w, t->w, sizeof(double) * (size_t)t->d_out * t->d_in);
  return 0;
}

/* proj/src/tile.cpp:103-119 */
int or_tile_set_weights(or_tile *t, const double *w) {
  const size_t n = (size_t)t->d_out * t->d_in;
  for (size_t c = 0; c < n; ++c) t->w[c] = cell_clip(t, c, w[c]);
  return 0;
}

int or_tile_get_device(const or_tile *t, double *dw_up, double *dw_down, double *w_max,
                       double *w_min) {
  const size_t n = (size_t)t->d_out * t->d_in;
  for (size_t c = 0; c < n; ++c) {
    if (dw_up) dw_up[c] = t->cells[6 * c + 0];
    if (dw_down) dw_down[c] = t->cells[6 * c + 1];
    if (w_max) w_max[c] = t->cells[6 * c + 2];
    if (w_min) w_min[c] = t->cells[6 * c + 3];
  }
  return 0;
}

/* proj/src/tile.cpp:158-169 */
int or_tile_apply_pulse_trains(or_tile *t, int bl, const uint8_t *xbits, const uint8_t *dbits,
                               const int *sign_x, const int *sign_d, int flip) {
  apply_coincidences(t, bl, xbits, dbits, sign_x, sign_d, flip);
  return 0;
}

/* proj/src/tile.cpp:128-156 */
int or_tile_apply_temporal_step(or_tile *t, const or_temporal_params *tp) {
  if (!(tp->decay_rate > 0.0 || tp->diffusion_sigma > 0.0 || tp->reset_prob > 0.0)) return 0;
  const size_t n = (size_t)t->d_out * t->d_in;
  for (size_t c = 0; c < n; ++c) {
    double w = t->w[c];
    if (tp->decay_rate > 0.0) {
      const double r = sclamp(tp->decay_rate * (1.0 + tp->decay_dtod * t->xi_decay[c]), 0.0, 1.0);
      w *= 1.0 - r;
    }
    if (tp->diffusion_sigma > 0.0) {
      const double sigma =
          smax(tp->diffusion_sigma * (1.0 + tp->diffusion_dtod * t->xi_diffusion[c]), 0.0);
      w += sigma * or_rng_gauss(&t->rng_temporal);
    }
    if (tp->reset_prob > 0.0) {
      const double p = sclamp(tp->reset_prob * (1.0 + tp->reset_dtod * t->xi_reset[c]), 0.0, 1.0);
      if (or_rng_bernoulli(&t->rng_temporal, p)) w = 0.0;
    }
    t->w[c] = cell_clip(t, c, w);
  }
  return 0;
}

/* proj/src/tile.cpp:171 */
int or_tile_end_minibatch(or_tile *t) { return or_tile_apply_temporal_step(t, &t->s.temporal); }

/* ======================================================================
 * TransferTile (Tiki-Taka) -- proj/src/compound.cpp:176-293
 * ====================================================================== */

struct or_transfer {
  int d_out, d_in;
  or_transfer_settings s;
  or_tile *fast, *slow;
  long counter, events;
  int next_column;
};

/* proj/src/compound.cpp:176-191 */
static int transfer_validate(const or_transfer_settings *s) {
  if (device_validate(&s->fast_device, "transfer.fast_device")) return -1;
  if (device_validate(&s->slow_device, "transfer.slow_device")) return -1;
  if (s->transfer_every < 0)
    return fail("transfer.transfer_every: must be >= 0 (0 disables transfer)");
  if (!(s->transfer_lr > 0.0)) return fail("transfer.transfer_lr: must be > 0");
  if (s->columns_per_event < 1) return fail("transfer.columns_per_event: must be >= 1");
  if (s->gamma < 0.0) return fail("transfer.gamma: must be >= 0");
  return 0;
}

/* proj/src/compound.cpp:31-42 */
static void member_settings(or_tile_settings *m, const or_device_params *dev,
                            const or_transfer_settings *s) {
  memset(m, 0, sizeof *m);
  m->device = *dev;
  m->forward_io = s->forward_io;
  m->backward_io = s->backward_io;
  m->update = s->update;
  m->temporal = s->temporal;
}

/* proj/src/compound.cpp:193-204 */
or_transfer *or_transfer_new(int d_out, int d_in, const or_transfer_settings *s, uint64_t seed) {
  or_tile_settings fs, ss;
  member_settings(&fs, &s->fast_device, s);
  member_settings(&ss, &s->slow_device, s);
  or_tile *fast = or_tile_new(d_out, d_in, &fs, derive_seed(seed, "fast"));
  if (!fast) return NULL;
  or_tile *slow = or_tile_new(d_out, d_in, &ss, derive_seed(seed, "slow"));
  if (!slow) {
    or_tile_free(fast);
    return NULL;
  }
  if (transfer_validate(s)) {
    or_tile_free(fast);
    or_tile_free(slow);
    return NULL;
  }
  or_transfer *t = (or_transfer *)calloc(1, sizeof(or_transfer));
  t->d_out = d_out;
  t->d_in = d_in;
  t->s = *s;
  t->fast = fast;
  t->slow = slow;
  return t;
}

void or_transfer_free(or_transfer *t) {
  if (!t) return;
  or_tile_free(t->fast);
  or_tile_free(t->slow);
  free(t);
}

/* proj/src/compound.cpp:206-215 */
int or_transfer_forward(or_transfer *t, const double *x, double *y) {
  if (or_tile_forward(t->slow, x, y)) return -1;
  if (t->s.gamma != 0.0) {
    double *ya = (double *)malloc(sizeof(double) * t->d_out);
    if (or_tile_forward(t->fast, x, ya)) {
      free(ya);
      return -1;
    }
    for (int i = 0; i < t->d_out; ++i) y[i] += t->s.gamma * ya[i];
    free(ya);
  }
  return 0;
}

/* proj/src/compound.cpp:217-226 */
int or_transfer_backward(or_transfer *t, const double *d, double *g) {
  if (or_tile_backward(t->slow, d, g)) return -1;
  if (t->s.gamma != 0.0) {
    double *ga = (double *)malloc(sizeof(double) * t->d_in);
    if (or_tile_backward(t->fast, d, ga)) {
      free(ga);
      return -1;
    }
    for (int j = 0; j < t->d_in; ++j) g[j] += t->s.gamma * ga[j];
    free(ga);
  }
  return 0;
}

/* proj/src/compound.cpp:257-267 */
int or_transfer_step(or_transfer *t) {
  double *onehot = (double *)calloc((size_t)t->d_in, sizeof(double));
  double *readout = (double *)malloc(sizeof(double) * t->d_out);
  onehot[t->next_column] = 1.0;
  const or_io_params *io = t->s.has_transfer_io ? &t->s.transfer_io : &t->s.forward_io;
  int rc = or_tile_forward_with_io(t->fast, onehot, io, readout);
  if (rc == 0 && max_abs(readout, t->d_out) > 0.0)
    rc = or_tile_update(t->slow, onehot, readout, t->s.transfer_lr);
  t->next_column = (t->next_column + 1) % t->d_in;
  free(onehot);
  free(readout);
  return rc;
}

/* proj/src/compound.cpp:247-255 */
static int tick(or_transfer *t) {
  ++t->counter;
  if (t->s.transfer_every > 0 && t->counter % t->s.transfer_every == 0) {
    ++t->events;
    for (int n = 0; n < t->s.columns_per_event; ++n)
      if (or_transfer_step(t)) return -1;
  }
  return 0;
}

/* proj/src/compound.cpp:240-245 */
int or_transfer_update(or_transfer *t, const double *x, const double *d, double lr) {
  if (or_tile_update(t->fast, x, d, lr)) return -1;
  if (!t->s.units_in_mbatch) return tick(t);
  return 0;
}

/* proj/src/compound.cpp:287-293 */
int or_transfer_end_minibatch(or_transfer *t) {
  if (t->s.units_in_mbatch && tick(t)) return -1;
  or_tile_end_minibatch(t->fast);
  or_tile_end_minibatch(t->slow);
  return 0;
}

/* proj/src/compound.cpp:269-280 */
int or_transfer_get_weights(const or_transfer *t, double *w) {
  or_tile_get_weights(t->slow, w);
  if (t->s.gamma != 0.0) {
    const size_t n = (size_t)t->d_out * t->d_in;
    for (size_t c = 0; c < n; ++c) w[c] += t->s.gamma * t->fast->w[c];
  }
  return 0;
}

/* proj/src/compound.cpp:282-285 */
int or_transfer_set_weights(or_transfer *t, const double *w) {
  or_tile_set_weights(t->slow, w);
  double *z = (double *)calloc((size_t)t->d_out * t->d_in, sizeof(double));
  or_tile_set_weights(t->fast, z);
  free(z);
  return 0;
}

long or_transfer_events(const or_transfer *t) { return t->events; }
or_tile *or_transfer_fast(or_transfer *t) { return t->fast; }
or_tile *or_transfer_slow(or_transfer *t) { return t->slow; }

/* ======================================================================
 * UnitCellTile -- proj/src/compound.cpp:12-174
 * ====================================================================== */

struct or_unitcell {
  int d_out, d_in;
  or_unitcell_settings s;
  or_tile *members[OR_MAX_CELL_DEVICES];
  int next_member; /* round-robin cursor, persists across mini-batches */
  or_rng rng_forward, rng_backward, rng_update;
  double *effective; /* [d_out * d_in], valid when !dirty */
  int dirty;
};

void or_default_unitcell_settings(or_unitcell_settings *s) {
  memset(s, 0, sizeof *s);
  s->n_devices = 1;
  or_default_device(&s->devices[0]);
  s->gains[0] = 1.0;
  s->policy = OR_UC_ALL_TOGETHER; /* compound.hpp:20 */
  or_default_io(&s->forward_io);
  or_default_io(&s->backward_io);
  or_default_update(&s->update);
  or_default_temporal(&s->temporal);
}

/* proj/src/compound.cpp:12-27 */
static int unitcell_validate(const or_unitcell_settings *s) {
  char buf[96];
  if (s->n_devices < 1) return fail("unit_cell.devices: need at least one device");
  if (s->n_devices > OR_MAX_CELL_DEVICES) return fail("unit_cell.gains: length must match devices");
  for (int k = 0; k < s->n_devices; ++k)
    if (!isfinite(s->gains[k])) return fail("unit_cell.gains: entries must be finite");
  for (int k = 0; k < s->n_devices; ++k) {
    snprintf(buf, sizeof buf, "unit_cell.devices[%d]", k);
    if (device_validate(&s->devices[k], buf)) return -1;
  }
  return 0;
}

/* proj/src/compound.cpp:46-48: member 0 shares the compound's seed */
static uint64_t member_seed(uint64_t seed, int k) {
  return k == 0 ? seed : derive_seed_idx(seed, "cell_member", (uint64_t)k);
}

/* proj/src/compound.cpp:52-64 */
or_unitcell *or_unitcell_new(int d_out, int d_in, const or_unitcell_settings *s, uint64_t seed) {
  if (unitcell_validate(s)) return NULL;
  or_unitcell *t = (or_unitcell *)calloc(1, sizeof(or_unitcell));
  t->d_out = d_out;
  t->d_in = d_in;
  t->s = *s;
  rng_init(&t->rng_forward, derive_seed(seed, "forward"));
  rng_init(&t->rng_backward, derive_seed(seed, "backward"));
  rng_init(&t->rng_update, derive_seed(seed, "update"));
  for (int k = 0; k < s->n_devices; ++k) {
    or_tile_settings m; /* compound.cpp:31-42 */
    memset(&m, 0, sizeof m);
    m.device = s->devices[k];
    m.forward_io = s->forward_io;
    m.backward_io = s->backward_io;
    m.update = s->update;
    m.temporal = s->temporal;
    t->members[k] = or_tile_new(d_out, d_in, &m, member_seed(seed, k));
    if (!t->members[k]) {
      or_unitcell_free(t);
      return NULL;
    }
  }
  t->effective = (double *)calloc((size_t)d_out * d_in, sizeof(double));
  t->dirty = 1;
  return t;
}

or_unitcell *or_unitcell_clone(const or_unitcell *t) {
  or_unitcell *c = (or_unitcell *)malloc(sizeof(or_unitcell));
  *c = *t;
  for (int k = 0; k < t->s.n_devices; ++k) c->members[k] = or_tile_clone(t->members[k]);
  c->effective = dup(t->effective, (size_t)t->d_out * t->d_in);
  return c;
}

void or_unitcell_free(or_unitcell *t) {
  if (!t) return;
  for (int k = 0; k < t->s.n_devices; ++k) or_tile_free(t->members[k]);
  free(t->effective);
  free(t);
}

/* proj/src/compound.cpp:66-80: sum_k g_k W_k, members in order */
static const double *effective(or_unitcell *t) {
  if (t->dirty) {
    const size_t n = (size_t)t->d_out * t->d_in;
    for (size_t c = 0; c < n; ++c) t->effective[c] = 0.0;
    for (int k = 0; k < t->s.n_devices; ++k) {
      const double g = t->s.gains[k], *w = t->members[k]->w;
      for (size_t c = 0; c < n; ++c) t->effective[c] += g * w[c];
    }
    t->dirty = 0;
  }
  return t->effective;
}

/* proj/src/compound.cpp:82-88 (the caller passes exactly d_in values) */
int or_unitcell_forward(or_unitcell *t, const double *x, double *y) {
  return or_analog_matvec(effective(t), t->d_out, t->d_in, x, &t->s.forward_io, &t->rng_forward,
                          0, y);
}

/* proj/src/compound.cpp:90-96 */
int or_unitcell_backward(or_unitcell *t, const double *d, double *g) {
  return or_analog_matvec(effective(t), t->d_out, t->d_in, d, &t->s.backward_io,
                          &t->rng_backward, 1, g);
}

/* proj/src/compound.cpp:98-107 */
int or_unitcell_forward_noisy(or_unitcell *t, const double *x, double extra_sigma, double *y) {
  or_io_params io;
  or_with_extra_weight_noise(&t->s.forward_io, extra_sigma, &io);
  return or_analog_matvec(effective(t), t->d_out, t->d_in, x, &io, &t->rng_forward, 0, y);
}

/* one translate + trains on the compound's update stream, applied to the
   members in `use` (proj/src/compound.cpp:118-146) */
static int unitcell_fire(or_unitcell *t, const double *x, const double *d, double lr,
                         double grain, int first, int last) {
  const int nr = t->d_out, nc = t->d_in;
  double *px = (double *)malloc(sizeof(double) * nc);
  double *pd = (double *)malloc(sizeof(double) * nr);
  int *sx = (int *)malloc(sizeof(int) * nc);
  int *sd = (int *)malloc(sizeof(int) * nr);
  int bl;
  int rc = or_translate(x, nc, d, nr, lr, grain, &t->s.update, &bl, px, pd, sx, sd);
  if (rc == 0) {
    uint8_t *xb = (uint8_t *)malloc((size_t)bl * nc + 1);
    uint8_t *db = (uint8_t *)malloc((size_t)bl * nr + 1);
    or_generate_trains(bl, px, nc, pd, nr, &t->rng_update, xb, db);
    for (int k = first; k <= last; ++k)
      if (t->s.gains[k] != 0.0)
        apply_coincidences(t->members[k], bl, xb, db, sx, sd, t->s.gains[k] < 0.0);
    free(xb);
    free(db);
  }
  free(px);
  free(pd);
  free(sx);
  free(sd);
  return rc;
}

/* proj/src/compound.cpp:109-147 */
int or_unitcell_update(or_unitcell *t, const double *x, const double *d, double lr) {
  if (lr == 0.0 || max_abs(x, t->d_in) == 0.0 || max_abs(d, t->d_out) == 0.0) return 0;
  t->dirty = 1;
  if (t->s.policy == OR_UC_ROUND_ROBIN) {
    const int k = t->next_member;
    t->next_member = (t->next_member + 1) % t->s.n_devices;
    const double grain = fabs(t->s.gains[k]) * t->members[k]->s.device.dw_min;
    if (grain == 0.0) return 0; /* zero-gain member: this event is a no-op */
    return unitcell_fire(t, x, d, lr, grain, k, k);
  }
  double grain = 0.0; /* all_together: sum_k |g_k| dw_min_k per coincidence */
  for (int k = 0; k < t->s.n_devices; ++k)
    grain += fabs(t->s.gains[k]) * t->members[k]->s.device.dw_min;
  if (grain == 0.0) return 0;
  return unitcell_fire(t, x, d, lr, grain, 0, t->s.n_devices - 1);
}

/* proj/src/compound.cpp:149 */
int or_unitcell_get_weights(const or_unitcell *t, double *w) {
  memcpy(w, effective((or_unitcell *)t), sizeof(double) * (size_t)t->d_out * t->d_in);
  return 0;
}

/* proj/src/compound.cpp:151-167 */
int or_unitcell_set_weights(or_unitcell *t, const double *w) {
  if (t->s.gains[0] == 0.0)
    return fail("set_weights: unit cell with zero first gain cannot be programmed");
  const size_t n = (size_t)t->d_out * t->d_in;
  double *scaled = (double *)calloc(n ? n : 1, sizeof(double));
  for (size_t c = 0; c < n; ++c) scaled[c] = w[c] / t->s.gains[0];
  or_tile_set_weights(t->members[0], scaled);
  for (size_t c = 0; c < n; ++c) scaled[c] = 0.0;
  for (int k = 1; k < t->s.n_devices; ++k) or_tile_set_weights(t->members[k], scaled);
  free(scaled);
  t->dirty = 1;
  return 0;
}

/* proj/src/compound.cpp:169-174 */
int or_unitcell_end_minibatch(or_unitcell *t) {
  for (int k = 0; k < t->s.n_devices; ++k) or_tile_end_minibatch(t->members[k]);
  t->dirty = 1;
  return 0;
}

int or_unitcell_n_members(const or_unitcell *t) { return t->s.n_devices; }
or_tile *or_unitcell_member(or_unitcell *t, int k) { return t->members[k]; }

/* ======================================================================
 * PCM inference -- proj/src/inference.cpp:14-110
 * ====================================================================== */

/* proj/src/inference.cpp:19-32 */
static int model_validate(const or_inference_model *m) {
  if (!(m->t0 > 0.0)) return fail("inference.t0: must be > 0");
  if (m->prog_noise_scale < 0.0 || m->read_noise_scale < 0.0 || m->nu_mean < 0.0 ||
      m->nu_std < 0.0)
    return fail("inference: noise scales and nu must be >= 0");
  if (m->nu_min < 0.0 || m->nu_max > 1.0 || m->nu_min > m->nu_max)
    return fail("inference: nu clip must satisfy 0 <= nu_min <= nu_max <= 1");
  if (m->compensation_probes < 1) return fail("inference.compensation_probes: must be >= 1");
  return 0;
}

/* proj/src/inference.cpp:14-17 */
static double prog_sigma(const or_inference_model *m, double w) {
  const double a = fabs(w);
  return m->prog_noise_scale * (m->prog_c0 + m->prog_c1 * a + m->prog_c2 * a * a);
}

/* proj/src/inference.cpp:34-61 */
int or_program(or_tile *t, const double *target, const or_inference_model *m, or_rng *rng,
               double *w0_out, double *nu_out) {
  if (model_validate(m)) return -1;
  const size_t n = (size_t)t->d_out * t->d_in;
  double *prog = (double *)calloc(n ? n : 1, sizeof(double));
  for (size_t c = 0; c < n; ++c) prog[c] = target[c] + prog_sigma(m, target[c]) * or_rng_gauss(rng);
  or_tile_set_weights(t, prog);
  free(prog);
  if (w0_out) memcpy(w0_out, t->w, sizeof(double) * n);
  for (size_t c = 0; c < n; ++c) {
    const double nu = m->nu_mean * (1.0 + m->nu_std * or_rng_gauss(rng));
    const double v = sclamp(nu, m->nu_min, m->nu_max);
    if (nu_out) nu_out[c] = v;
  }
  return 0;
}

/* proj/src/inference.cpp:63-76 */
int or_drift_to(or_tile *t, const double *w0, const double *nu, double t0, double time_s) {
  if (time_s < t0) return fail("drift_to: t < t0");
  const double ratio = time_s / t0;
  const size_t n = (size_t)t->d_out * t->d_in;
  double *w = (double *)malloc(sizeof(double) * n);
  for (size_t c = 0; c < n; ++c) w[c] = w0[c] * pow(ratio, -nu[c]);
  or_tile_set_weights(t, w);
  free(w);
  return 0;
}

/* proj/src/inference.cpp:85-95 */
int or_probe_readout(or_tile *t, const or_inference_model *m, double *out) {
  double *probe = (double *)malloc(sizeof(double) * t->d_in);
  double *y = (double *)malloc(sizeof(double) * t->d_out);
  for (int j = 0; j < t->d_in; ++j) probe[j] = 1.0;
  double acc = 0.0;
  int rc = 0;
  for (int r = 0; r < m->compensation_probes && rc == 0; ++r) {
    rc = or_tile_forward_noisy(t, probe, m->read_noise_scale, y);
    for (int i = 0; i < t->d_out && rc == 0; ++i) acc += fabs(y[i]);
  }
  free(probe);
  free(y);
  *out = acc / m->compensation_probes;
  return rc;
}

/* proj/src/inference.cpp:103-110 */
int or_drift_compensation_factor(or_tile *t, double baseline, const or_inference_model *m,
                                 double *alpha) {
  double current;
  if (or_probe_readout(t, m, &current)) return -1;
  if (current <= 1e-12)
    return fail("drift_compensation_factor: degenerate readout (all-zero tile?)");
  *alpha = baseline / current;
  return 0;
}
