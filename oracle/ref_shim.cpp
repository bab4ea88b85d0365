// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" adapter that exposes the REFERENCE implementation (xbarsim,
// compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libxbref.so) through the same C API as the plain-C
// restatement (oracle/oracle.h).  It contains no algorithm of its own: each
// entry point converts the POD structs into the reference's settings structs
// and calls the reference function named in the comment.  Its only purpose is
// to pin oracle/xbarsim_oracle.c (tests/test_oracle_pin.py) and to generate
// the golden fixtures under tests/golden/.
#include "oracle.h"

#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "xbarsim/compound.hpp"
#include "xbarsim/device.hpp"
#include "xbarsim/inference.hpp"
#include "xbarsim/io.hpp"
#include "xbarsim/pulsed.hpp"
#include "xbarsim/rng.hpp"
#include "xbarsim/tile.hpp"

using namespace xbarsim;

namespace {

thread_local std::string g_err;

template <class F> int guard(F &&f) {
  try {
    f();
    return 0;
  } catch (const std::exception &e) {
    g_err = e.what();
    return -1;
  }
}

DeviceParams to_ref(const or_device_params &p) {
  DeviceParams d;
  d.kind = static_cast<DeviceKind>(p.kind);
  d.dw_min = p.dw_min;
  d.dw_min_dtod = p.dw_min_dtod;
  d.dw_min_std = p.dw_min_std;
  d.up_down = p.up_down;
  d.up_down_dtod = p.up_down_dtod;
  d.w_max = p.w_max;
  d.w_min = p.w_min;
  d.w_max_dtod = p.w_max_dtod;
  d.w_min_dtod = p.w_min_dtod;
  d.slope = p.slope;
  d.gamma = p.gamma;
  return d;
}

void from_ref(const DeviceParams &d, or_device_params *p) {
  std::memset(p, 0, sizeof *p);
  p->kind = static_cast<int>(d.kind);
  p->dw_min = d.dw_min;
  p->dw_min_dtod = d.dw_min_dtod;
  p->dw_min_std = d.dw_min_std;
  p->up_down = d.up_down;
  p->up_down_dtod = d.up_down_dtod;
  p->w_max = d.w_max;
  p->w_min = d.w_min;
  p->w_max_dtod = d.w_max_dtod;
  p->w_min_dtod = d.w_min_dtod;
  p->slope = d.slope;
  p->gamma = d.gamma;
}

IOParams to_ref(const or_io_params &p) {
  IOParams io;
  io.dac_bits = p.dac_bits;
  io.adc_bits = p.adc_bits;
  io.input_bound = p.input_bound;
  io.output_bound = p.output_bound;
  io.sigma_inp = p.sigma_inp;
  io.sigma_out = p.sigma_out;
  io.sigma_w = p.sigma_w;
  io.noise_management = static_cast<NoiseManagement>(p.noise_management);
  io.is_perfect = p.is_perfect != 0;
  return io;
}

void from_ref(const IOParams &io, or_io_params *p) {
  std::memset(p, 0, sizeof *p);
  p->dac_bits = io.dac_bits;
  p->adc_bits = io.adc_bits;
  p->input_bound = io.input_bound;
  p->output_bound = io.output_bound;
  p->sigma_inp = io.sigma_inp;
  p->sigma_out = io.sigma_out;
  p->sigma_w = io.sigma_w;
  p->noise_management = static_cast<int>(io.noise_management);
  p->is_perfect = io.is_perfect ? 1 : 0;
}

UpdateParams to_ref(const or_update_params &p) {
  UpdateParams u;
  u.bl = p.bl;
  u.bl_management = p.bl_management != 0;
  u.pulse_type = static_cast<PulseType>(p.pulse_type);
  return u;
}

TemporalParams to_ref(const or_temporal_params &p) {
  TemporalParams t;
  t.decay_rate = p.decay_rate;
  t.decay_dtod = p.decay_dtod;
  t.diffusion_sigma = p.diffusion_sigma;
  t.diffusion_dtod = p.diffusion_dtod;
  t.reset_prob = p.reset_prob;
  t.reset_dtod = p.reset_dtod;
  return t;
}

TileSettings to_ref(const or_tile_settings &s) {
  TileSettings t;
  t.device = to_ref(s.device);
  t.forward_io = to_ref(s.forward_io);
  t.backward_io = to_ref(s.backward_io);
  t.update = to_ref(s.update);
  t.temporal = to_ref(s.temporal);
  return t;
}

TransferSettings to_ref(const or_transfer_settings &s) {
  TransferSettings t;
  t.fast_device = to_ref(s.fast_device);
  t.slow_device = to_ref(s.slow_device);
  t.forward_io = to_ref(s.forward_io);
  t.backward_io = to_ref(s.backward_io);
  t.update = to_ref(s.update);
  t.temporal = to_ref(s.temporal);
  t.transfer_every = s.transfer_every;
  t.units_in_mbatch = s.units_in_mbatch != 0;
  t.transfer_lr = s.transfer_lr;
  t.columns_per_event = s.columns_per_event;
  t.gamma = s.gamma;
  if (s.has_transfer_io) t.transfer_io = to_ref(s.transfer_io);
  return t;
}

UnitCellSettings to_ref(const or_unitcell_settings &s) {
  UnitCellSettings u;
  for (int k = 0; k < s.n_devices && k < OR_MAX_CELL_DEVICES; ++k) {
    u.devices.push_back(to_ref(s.devices[k]));
    u.gains.push_back(s.gains[k]);
  }
  u.policy = s.policy == OR_UC_ROUND_ROBIN ? UnitCellPolicy::round_robin
                                           : UnitCellPolicy::all_together;
  u.forward_io = to_ref(s.forward_io);
  u.backward_io = to_ref(s.backward_io);
  u.update = to_ref(s.update);
  u.temporal = to_ref(s.temporal);
  return u;
}

InferenceNoiseModel to_ref(const or_inference_model &m) {
  InferenceNoiseModel r;
  r.prog_noise_scale = m.prog_noise_scale;
  r.prog_c0 = m.prog_c0;
  r.prog_c1 = m.prog_c1;
  r.prog_c2 = m.prog_c2;
  r.read_noise_scale = m.read_noise_scale;
  r.nu_mean = m.nu_mean;
  r.nu_std = m.nu_std;
  r.t0 = m.t0;
  r.nu_min = m.nu_min;
  r.nu_max = m.nu_max;
  r.compensation_probes = m.compensation_probes;
  return r;
}

Matrix to_matrix(const double *w, int rows, int cols) {
  Matrix m(rows, cols);
  std::memcpy(m.data(), w, sizeof(double) * m.size());
  return m;
}

void copy_out(const std::vector<double> &v, double *out) {
  std::memcpy(out, v.data(), sizeof(double) * v.size());
}

} // namespace

struct or_rng {
  RngStream r;
};
struct or_tile {
  // owned tiles hold `own`; member tiles of a transfer compound borrow `ptr`
  std::unique_ptr<AnalogTile> own;
  AnalogTile *ptr = nullptr;
  AnalogTile &t() { return *ptr; }
};
struct or_transfer {
  std::unique_ptr<TransferTile> t;
  or_tile fast, slow;
};
struct or_unitcell {
  std::unique_ptr<UnitCellTile> t;
  or_tile members[OR_MAX_CELL_DEVICES];
  void bind() {
    for (int k = 0; k < t->n_members(); ++k)
      members[k].ptr = const_cast<AnalogTile *>(&t->member(k));
  }
};

extern "C" {

const char *or_last_error(void) { return g_err.c_str(); }
const char *or_impl_name(void) { return "reference"; }

void or_default_device(or_device_params *p) { from_ref(DeviceParams{}, p); }
void or_default_io(or_io_params *p) { from_ref(IOParams{}, p); }
void or_perfect_io(or_io_params *p) { from_ref(perfect_io(), p); }
void or_default_update(or_update_params *p) {
  UpdateParams u;
  p->bl = u.bl;
  p->bl_management = u.bl_management;
  p->pulse_type = static_cast<int>(u.pulse_type);
}
void or_default_temporal(or_temporal_params *p) { std::memset(p, 0, sizeof *p); }
void or_default_tile_settings(or_tile_settings *s) {
  std::memset(s, 0, sizeof *s);
  or_default_device(&s->device);
  or_default_io(&s->forward_io);
  or_default_io(&s->backward_io);
  or_default_update(&s->update);
}
void or_default_transfer_settings(or_transfer_settings *s) {
  std::memset(s, 0, sizeof *s);
  TransferSettings r;
  from_ref(r.fast_device, &s->fast_device);
  from_ref(r.slow_device, &s->slow_device);
  from_ref(r.forward_io, &s->forward_io);
  from_ref(r.backward_io, &s->backward_io);
  or_default_update(&s->update);
  s->transfer_every = r.transfer_every;
  s->units_in_mbatch = r.units_in_mbatch;
  s->transfer_lr = r.transfer_lr;
  s->columns_per_event = r.columns_per_event;
  s->gamma = r.gamma;
  s->has_transfer_io = 0;
  from_ref(IOParams{}, &s->transfer_io);
}
void or_default_inference_model(or_inference_model *m) {
  InferenceNoiseModel r;
  std::memset(m, 0, sizeof *m);
  m->prog_noise_scale = r.prog_noise_scale;
  m->prog_c0 = r.prog_c0;
  m->prog_c1 = r.prog_c1;
  m->prog_c2 = r.prog_c2;
  m->read_noise_scale = r.read_noise_scale;
  m->nu_mean = r.nu_mean;
  m->nu_std = r.nu_std;
  m->t0 = r.t0;
  m->nu_min = r.nu_min;
  m->nu_max = r.nu_max;
  m->compensation_probes = r.compensation_probes;
}
int or_device_preset(const char *name, or_device_params *p) {
  return guard([&] { from_ref(device_preset(name), p); });
}

or_rng *or_rng_new(uint64_t seed) { return new or_rng{RngStream(seed)}; }
or_rng *or_rng_derive(const or_rng *r, const char *name) { return new or_rng{r->r.derive(name)}; }
or_rng *or_rng_derive_idx(const or_rng *r, const char *name, uint64_t index) {
  return new or_rng{r->r.derive(name, index)};
}
void or_rng_free(or_rng *r) { delete r; }
uint64_t or_rng_base_seed(const or_rng *r) { return r->r.base_seed(); }
uint64_t or_rng_next_u64(or_rng *r) { return r->r.next_u64(); }
double or_rng_uniform(or_rng *r) { return r->r.uniform(); }
double or_rng_gauss(or_rng *r) { return r->r.gauss(); }
int or_rng_bernoulli(or_rng *r, double p) { return r->r.bernoulli(p) ? 1 : 0; }

double or_quantize_uniform(double v, double bound, int bits) {
  return quantize_uniform(v, bound, bits);
}
void or_with_extra_weight_noise(const or_io_params *io, double extra, or_io_params *out) {
  from_ref(with_extra_weight_noise(to_ref(*io), extra), out);
}
int or_analog_matvec(const double *w, int rows, int cols, const double *in,
                     const or_io_params *io, or_rng *rng, int transposed, double *out) {
  return guard([&] {
    Matrix m = to_matrix(w, rows, cols);
    const int n = transposed ? rows : cols;
    copy_out(analog_matvec(m, std::span<const double>(in, n), to_ref(*io), rng->r, transposed != 0),
             out);
  });
}

int or_realize_cell(const or_device_params *p, or_rng *rng, double *cell) {
  return guard([&] {
    DeviceRealization c = realize_cell(to_ref(*p), rng->r);
    cell[0] = c.dw_min_up;
    cell[1] = c.dw_min_down;
    cell[2] = c.w_max;
    cell[3] = c.w_min;
    cell[4] = c.slope;
    cell[5] = c.gamma;
  });
}
double or_apply_pulse(const double *cell, double w, int up, int kind, double dw_min_std,
                      or_rng *rng) {
  DeviceRealization c;
  c.dw_min_up = cell[0];
  c.dw_min_down = cell[1];
  c.w_max = cell[2];
  c.w_min = cell[3];
  c.slope = cell[4];
  c.gamma = cell[5];
  return apply_pulse(c, w, up ? PulseDirection::up : PulseDirection::down,
                     static_cast<DeviceKind>(kind), dw_min_std, rng->r);
}

int or_translate(const double *x, int nx, const double *d, int nd, double lr, double dw_min,
                 const or_update_params *up, int *bl, double *px, double *pd, int *sx, int *sd) {
  return guard([&] {
    PulsePlan p = translate(std::span<const double>(x, nx), std::span<const double>(d, nd), lr,
                            dw_min, to_ref(*up));
    *bl = p.bl;
    copy_out(p.prob_x, px);
    copy_out(p.prob_d, pd);
    std::memcpy(sx, p.sign_x.data(), sizeof(int) * nx);
    std::memcpy(sd, p.sign_d.data(), sizeof(int) * nd);
  });
}
int or_generate_trains(int bl, const double *px, int nx, const double *pd, int nd, or_rng *rng,
                       uint8_t *xbits, uint8_t *dbits) {
  return guard([&] {
    PulsePlan p;
    p.bl = bl;
    p.prob_x.assign(px, px + nx);
    p.prob_d.assign(pd, pd + nd);
    p.sign_x.assign(nx, 1);
    p.sign_d.assign(nd, 1);
    PulseTrains tr = generate_trains(p, rng->r);
    std::memcpy(xbits, tr.x_bits.data(), tr.x_bits.size());
    std::memcpy(dbits, tr.d_bits.data(), tr.d_bits.size());
  });
}

or_tile *or_tile_new(int d_out, int d_in, const or_tile_settings *s, uint64_t seed) {
  or_tile *t = nullptr;
  guard([&] {
    auto own = std::make_unique<AnalogTile>(d_out, d_in, to_ref(*s), seed);
    t = new or_tile;
    t->ptr = own.get();
    t->own = std::move(own);
  });
  return t;
}
or_tile *or_tile_clone(const or_tile *src) {
  auto *t = new or_tile;
  t->own = std::make_unique<AnalogTile>(*src->ptr);
  t->ptr = t->own.get();
  return t;
}
void or_tile_free(or_tile *t) { delete t; }

int or_tile_forward(or_tile *t, const double *x, double *y) {
  return guard([&] {
    copy_out(t->t().forward(std::span<const double>(x, t->t().d_in())), y);
  });
}
int or_tile_backward(or_tile *t, const double *d, double *g) {
  return guard([&] {
    copy_out(t->t().backward(std::span<const double>(d, t->t().d_out())), g);
  });
}
int or_tile_update(or_tile *t, const double *x, const double *d, double lr) {
  return guard([&] {
    t->t().update(std::span<const double>(x, t->t().d_in()),
                  std::span<const double>(d, t->t().d_out()), lr);
  });
}
int or_tile_forward_noisy(or_tile *t, const double *x, double extra_sigma, double *y) {
  return guard([&] {
    copy_out(t->t().forward_noisy(std::span<const double>(x, t->t().d_in()), extra_sigma), y);
  });
}
int or_tile_forward_with_io(or_tile *t, const double *x, const or_io_params *io, double *y) {
  return guard([&] {
    copy_out(t->t().forward_with_io(std::span<const double>(x, t->t().d_in()), to_ref(*io)), y);
  });
}
int or_tile_get_weights(const or_tile *t, double *w) {
  Matrix m = t->ptr->get_weights();
  std::memcpy(w, m.data(), sizeof(double) * m.size());
  return 0;
}
int or_tile_set_weights(or_tile *t, const double *w) {
  return guard([&] { t->t().set_weights(to_matrix(w, t->t().d_out(), t->t().d_in())); });
}
int or_tile_get_device(const or_tile *t, double *dw_up, double *dw_down, double *w_max,
                       double *w_min) {
  const DeviceMatrix &dev = t->ptr->device();
  size_t c = 0;
  for (int i = 0; i < dev.rows(); ++i) {
    for (int j = 0; j < dev.cols(); ++j, ++c) {
      const DeviceRealization &r = dev.at(i, j);
      if (dw_up) dw_up[c] = r.dw_min_up;
      if (dw_down) dw_down[c] = r.dw_min_down;
      if (w_max) w_max[c] = r.w_max;
      if (w_min) w_min[c] = r.w_min;
    }
  }
  return 0;
}
int or_tile_apply_pulse_trains(or_tile *t, int bl, const uint8_t *xbits, const uint8_t *dbits,
                               const int *sign_x, const int *sign_d, int flip) {
  return guard([&] {
    PulseTrains tr;
    tr.bl = bl;
    tr.x_lines = t->t().d_in();
    tr.d_lines = t->t().d_out();
    tr.x_bits.assign(xbits, xbits + static_cast<size_t>(bl) * tr.x_lines);
    tr.d_bits.assign(dbits, dbits + static_cast<size_t>(bl) * tr.d_lines);
    t->t().apply_pulse_trains(tr, std::span<const int>(sign_x, tr.x_lines),
                              std::span<const int>(sign_d, tr.d_lines), flip != 0);
  });
}
int or_tile_apply_temporal_step(or_tile *t, const or_temporal_params *tp) {
  return guard([&] { t->t().apply_temporal_step(to_ref(*tp)); });
}
int or_tile_end_minibatch(or_tile *t) {
  return guard([&] { t->t().end_minibatch(); });
}

or_transfer *or_transfer_new(int d_out, int d_in, const or_transfer_settings *s, uint64_t seed) {
  or_transfer *t = nullptr;
  guard([&] {
    auto tt = std::make_unique<TransferTile>(d_out, d_in, to_ref(*s), seed);
    t = new or_transfer;
    t->t = std::move(tt);
    t->fast.ptr = &t->t->fast_tile();
    t->slow.ptr = &t->t->slow_tile();
  });
  return t;
}
void or_transfer_free(or_transfer *t) { delete t; }
int or_transfer_forward(or_transfer *t, const double *x, double *y) {
  return guard([&] { copy_out(t->t->forward(std::span<const double>(x, t->t->d_in())), y); });
}
int or_transfer_backward(or_transfer *t, const double *d, double *g) {
  return guard([&] { copy_out(t->t->backward(std::span<const double>(d, t->t->d_out())), g); });
}
int or_transfer_update(or_transfer *t, const double *x, const double *d, double lr) {
  return guard([&] {
    t->t->update(std::span<const double>(x, t->t->d_in()),
                 std::span<const double>(d, t->t->d_out()), lr);
  });
}
int or_transfer_end_minibatch(or_transfer *t) {
  return guard([&] { t->t->end_minibatch(); });
}
int or_transfer_step(or_transfer *t) {
  return guard([&] { t->t->transfer_step(); });
}
int or_transfer_get_weights(const or_transfer *t, double *w) {
  Matrix m = t->t->get_weights();
  std::memcpy(w, m.data(), sizeof(double) * m.size());
  return 0;
}
int or_transfer_set_weights(or_transfer *t, const double *w) {
  return guard([&] { t->t->set_weights(to_matrix(w, t->t->d_out(), t->t->d_in())); });
}
long or_transfer_events(const or_transfer *t) { return t->t->transfer_events(); }
or_tile *or_transfer_fast(or_transfer *t) { return &t->fast; }
or_tile *or_transfer_slow(or_transfer *t) { return &t->slow; }

void or_default_unitcell_settings(or_unitcell_settings *s) {
  std::memset(s, 0, sizeof *s);
  UnitCellSettings r;
  s->n_devices = 1;
  from_ref(DeviceParams{}, &s->devices[0]);
  s->gains[0] = 1.0;
  s->policy = r.policy == UnitCellPolicy::round_robin ? OR_UC_ROUND_ROBIN : OR_UC_ALL_TOGETHER;
  from_ref(r.forward_io, &s->forward_io);
  from_ref(r.backward_io, &s->backward_io);
  or_default_update(&s->update);
}
or_unitcell *or_unitcell_new(int d_out, int d_in, const or_unitcell_settings *s, uint64_t seed) {
  or_unitcell *t = nullptr;
  guard([&] {
    auto u = std::make_unique<UnitCellTile>(d_out, d_in, to_ref(*s), seed);
    t = new or_unitcell;
    t->t = std::move(u);
    t->bind();
  });
  return t;
}
or_unitcell *or_unitcell_clone(const or_unitcell *src) {
  auto *t = new or_unitcell;
  t->t = std::make_unique<UnitCellTile>(*src->t);
  t->bind();
  return t;
}
void or_unitcell_free(or_unitcell *t) { delete t; }
int or_unitcell_forward(or_unitcell *t, const double *x, double *y) {
  return guard([&] { copy_out(t->t->forward(std::span<const double>(x, t->t->d_in())), y); });
}
int or_unitcell_backward(or_unitcell *t, const double *d, double *g) {
  return guard([&] { copy_out(t->t->backward(std::span<const double>(d, t->t->d_out())), g); });
}
int or_unitcell_forward_noisy(or_unitcell *t, const double *x, double extra, double *y) {
  return guard([&] {
    copy_out(t->t->forward_noisy(std::span<const double>(x, t->t->d_in()), extra), y);
  });
}
int or_unitcell_update(or_unitcell *t, const double *x, const double *d, double lr) {
  return guard([&] {
    t->t->update(std::span<const double>(x, t->t->d_in()),
                 std::span<const double>(d, t->t->d_out()), lr);
  });
}
int or_unitcell_get_weights(const or_unitcell *t, double *w) {
  Matrix m = t->t->get_weights();
  std::memcpy(w, m.data(), sizeof(double) * m.size());
  return 0;
}
int or_unitcell_set_weights(or_unitcell *t, const double *w) {
  return guard([&] { t->t->set_weights(to_matrix(w, t->t->d_out(), t->t->d_in())); });
}
int or_unitcell_end_minibatch(or_unitcell *t) {
  return guard([&] { t->t->end_minibatch(); });
}
int or_unitcell_n_members(const or_unitcell *t) { return t->t->n_members(); }
or_tile *or_unitcell_member(or_unitcell *t, int k) { return &t->members[k]; }

int or_program(or_tile *t, const double *target, const or_inference_model *m, or_rng *rng,
               double *w0_out, double *nu_out) {
  return guard([&] {
    ProgrammedState st =
        program(t->t(), to_matrix(target, t->t().d_out(), t->t().d_in()), to_ref(*m), rng->r);
    if (w0_out) std::memcpy(w0_out, st.w0.data(), sizeof(double) * st.w0.size());
    if (nu_out) std::memcpy(nu_out, st.nu.data(), sizeof(double) * st.nu.size());
  });
}
int or_drift_to(or_tile *t, const double *w0, const double *nu, double t0, double time_s) {
  return guard([&] {
    ProgrammedState st;
    st.w0 = to_matrix(w0, t->t().d_out(), t->t().d_in());
    st.nu = to_matrix(nu, t->t().d_out(), t->t().d_in());
    st.t0 = t0;
    st.t = t0;
    drift_to(t->t(), st, time_s);
  });
}
int or_probe_readout(or_tile *t, const or_inference_model *m, double *out) {
  return guard([&] { *out = calibrate_compensation(t->t(), to_ref(*m)).baseline_readout; });
}
int or_drift_compensation_factor(or_tile *t, double baseline, const or_inference_model *m,
                                 double *alpha) {
  return guard([&] {
    *alpha = drift_compensation_factor(t->t(), DriftCompensation{baseline}, to_ref(*m));
  });
}

} // extern "C"
