// capi.cu -- the C ABI of librtucker_b200.so (include/rtucker.h, include/rtucker_b200.h).
//
// Handle/ownership/error semantics follow ref capi.cpp:20-73: opaque heap
// handles, NULL-argument checks before any work, exceptions mapped to status
// codes in one place (`guarded`), message in a thread-local last error.
// All arithmetic runs on the GPU through engine.cu; there is no CPU path.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <memory>
#include <new>
#include <sstream>
#include <string>
#include <unordered_set>
#include <vector>

// the C ABI is the only exported surface (the .so is built -fvisibility=hidden)
#pragma GCC visibility push(default)
#include "../../include/rtucker.h"
#include "../../include/rtucker_b200.h"
#pragma GCC visibility pop
#include "engine.h"

struct rtucker_tensor {
  std::vector<uint64_t> shape;
  // Two copies, each materialised on demand: tensors created from host data are
  // uploaded (and checked) at creation when a GPU is present, and the host copy is only
  // downloaded again if rtucker_tensor_data / rtucker_tensor_write ask for it.
  mutable std::vector<double> host;
  mutable bool host_valid = true;
  mutable rtb::DevBuf dev;
  mutable bool dev_valid = false;
  uint64_t size() const {
    uint64_t s = 1;
    for (auto v : shape) s *= v;
    return s;
  }
  const double* device() const {
    if (!dev_valid) {
      cudaStream_t st = rtb::current_stream();
      dev.ensure(size() * 8, st);
      RTB_CUDA(cudaMemcpyAsync(dev.p, host.data(), size() * 8, cudaMemcpyHostToDevice, st));
      dev_valid = true;
    }
    return dev.as<double>();
  }
  const double* host_data() const {
    if (!host_valid) {
      cudaStream_t st = rtb::current_stream();
      host.resize(size());
      RTB_CUDA(cudaMemcpyAsync(host.data(), dev.p, size() * 8, cudaMemcpyDeviceToHost, st));
      RTB_CUDA(cudaStreamSynchronize(st));
      host_valid = true;
    }
    return host.data();
  }
};

struct rtucker_model {
  std::vector<uint64_t> shape, ranks;
  std::vector<double> core, factors;
  double lambda = 0.0;
};

struct rtucker_als_result {
  rtb::AlsOutput out;
};

namespace {

thread_local std::string g_last_error;

rtucker_status fail(rtucker_status code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

template <typename Fn>
rtucker_status guarded(Fn&& fn) {
  try {
    fn();
    return RTUCKER_OK;
  } catch (const rtb::Error& e) {
    return fail(static_cast<rtucker_status>(e.code), e.what());
  } catch (const std::invalid_argument& e) {
    return fail(RTUCKER_ERR_INVALID_ARGUMENT, e.what());
  } catch (const std::bad_alloc&) {
    return fail(RTUCKER_ERR_UNKNOWN, "out of memory");
  } catch (const std::runtime_error& e) {  // file problems (ref capi.cpp:52-53)
    return fail(RTUCKER_ERR_IO, e.what());
  } catch (const std::exception& e) {
    return fail(RTUCKER_ERR_UNKNOWN, e.what());
  }
}

rtucker_status copy_label(const std::string& label, char* buf, size_t len) {
  if (buf == nullptr || len == 0 || label.size() + 1 > len)
    return fail(RTUCKER_ERR_INVALID_ARGUMENT, "step buffer too small");
  std::memcpy(buf, label.c_str(), label.size() + 1);
  return RTUCKER_OK;
}

// ref tensor.cpp:7-20, 32-42
uint64_t checked_volume(const uint64_t* shape, uint32_t order) {
  if (order == 0 || order > 8) throw rtb::Error(1, "DenseTensor: order must be in [1, 8]");
  uint64_t v = 1;
  for (uint32_t n = 0; n < order; ++n) {
    if (shape[n] == 0) throw rtb::Error(1, "DenseTensor: zero-length dimension");
    if (v > UINT64_MAX / shape[n]) throw rtb::Error(1, "DenseTensor: shape overflow");
    v *= shape[n];
  }
  return v;
}

void check_finite(const double* v, uint64_t n, const char* what) {
  for (uint64_t i = 0; i < n; ++i)
    if (!std::isfinite(v[i])) throw rtb::Error(1, std::string(what) + ": non-finite entry");
}

rtb::AlsOptions to_options(const rtucker_als_options* o) {
  rtb::AlsOptions a;
  a.lambda = o->lambda;
  a.sketched = o->sketched_core != 0;
  a.epsilon = o->epsilon;
  a.delta = o->delta;
  a.seed = o->seed;
  a.max_iterations = o->max_iterations;
  a.tolerance = o->tolerance;
  a.sample_override = o->sample_count_override;
  a.record_history = o->record_history != 0;
  return a;
}

rtucker_model* model_from_output(const rtb::AlsOutput& o) {
  auto* m = new rtucker_model;
  m->shape = o.shape;
  m->ranks = o.ranks;
  m->core = o.core;
  m->factors = o.factors;
  m->lambda = o.lambda;
  return m;
}

// SplitMix64 stream (ref rng.hpp:12-62), host side for the synthetic generator.
struct Rng {
  uint64_t s;
  bool have = false;
  double spare = 0.0;
  uint64_t u64() { return rtb::sm_mix(s += rtb::kGamma); }
  double unit() { return (double)(u64() >> 11) * 0x1.0p-53; }
  uint64_t below(uint64_t b) {
    const uint64_t thr = (0 - b) % b;
    for (;;) {
      const uint64_t r = u64();
      if (r >= thr) return r % b;
    }
  }
  double normal() {
    if (have) {
      have = false;
      return spare;
    }
    double u1 = unit(), u2 = unit();
    while (u1 <= 0.0) u1 = unit();
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double angle = 6.283185307179586476925286766559 * u2;
    spare = radius * std::sin(angle);
    have = true;
    return radius * std::cos(angle);
  }
};

uint64_t fnv1a(const void* data, size_t bytes, uint64_t h) {
  const auto* p = static_cast<const unsigned char*>(data);
  for (size_t i = 0; i < bytes; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

template <typename T>
void wr(std::ofstream& o, T v) {
  o.write(reinterpret_cast<const char*>(&v), sizeof(T));
}
template <typename T>
T rd(std::ifstream& i, const std::string& what) {
  T v;
  i.read(reinterpret_cast<char*>(&v), sizeof(T));
  if (!i) throw std::runtime_error(what);
  return v;
}

}  // namespace

extern "C" {

const char* rtucker_version(void) { return "1.0.0"; }
const char* rtucker_last_error(void) { return g_last_error.c_str(); }

rtucker_status rtucker_tensor_create(const uint64_t* shape, uint32_t order, const double* data,
                                     rtucker_tensor** out) {
  if (!shape || !data || !out) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    const uint64_t v = checked_volume(shape, order);
    auto t = std::make_unique<rtucker_tensor>();
    t->shape.assign(shape, shape + order);
    if (rtb::cuda_device_present()) {
      // the copy the reference makes (ref tensor.cpp:32-42) goes straight to HBM
      cudaStream_t st = rtb::current_stream();
      t->dev.ensure(v * 8, st);
      rtb::upload_checked(t->dev.as<double>(), data, v, st, "DenseTensor");
      t->dev_valid = true;
      t->host_valid = false;
    } else {
      check_finite(data, v, "DenseTensor");
      t->host.assign(data, data + v);
    }
    *out = t.release();
  });
}

rtucker_status rtucker_tensor_read(const char* path, rtucker_tensor** out) {
  if (!path || !out) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    // DTEN1 (ref tensor_io.cpp:54-89): "DTEN", u8 version 1, u32 order, u64 dims, f64 data LE
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error(std::string("read_tensor: cannot open ") + path);
    char magic[4];
    in.read(magic, 4);
    if (!in || std::memcmp(magic, "DTEN", 4) != 0)
      throw std::runtime_error(std::string("read_tensor: bad magic in ") + path);
    if (rd<uint8_t>(in, "read_tensor: truncated version") != 1)
      throw std::runtime_error("read_tensor: unsupported version");
    const uint32_t order = rd<uint32_t>(in, "read_tensor: truncated order");
    if (order == 0 || order > 8) throw std::runtime_error("read_tensor: order outside [1, 8]");
    std::vector<uint64_t> shape(order);
    uint64_t vol = 1;
    for (uint32_t n = 0; n < order; ++n) {
      const uint64_t dim = rd<uint64_t>(in, "read_tensor: truncated shape");
      if (dim == 0 || dim > UINT64_MAX / vol) throw std::runtime_error("read_tensor: shape overflow");
      shape[n] = dim;
      vol *= dim;
    }
    auto t = std::make_unique<rtucker_tensor>();
    t->host.resize(vol);
    in.read(reinterpret_cast<char*>(t->host.data()), (std::streamsize)(vol * 8));
    if (!in || (uint64_t)in.gcount() != vol * 8)
      throw std::runtime_error(std::string("read_tensor: truncated payload in ") + path);
    check_finite(t->host.data(), vol, "DenseTensor");
    t->shape = shape;
    *out = t.release();
  });
}

rtucker_status rtucker_tensor_read_csv(const char* path, rtucker_tensor** out) {
  if (!path || !out) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    // coordinate CSV: i_1,...,i_N,value per line; '#' comments (ref tensor_io.cpp:91-142)
    std::ifstream in(path);
    if (!in) throw std::runtime_error(std::string("read_tensor_csv: cannot open ") + path);
    std::vector<std::vector<uint64_t>> idx;
    std::vector<double> vals;
    std::vector<uint64_t> shape;
    std::string line;
    size_t ln = 0;
    while (std::getline(in, line)) {
      ++ln;
      if (line.empty() || line[0] == '#') continue;
      std::stringstream ss(line);
      std::vector<double> f;
      std::string field;
      while (std::getline(ss, field, ',')) f.push_back(std::stod(field));
      if (f.size() < 2)
        throw std::runtime_error("read_tensor_csv: line " + std::to_string(ln) +
                                 " needs at least one index and a value");
      std::vector<uint64_t> ix(f.size() - 1);
      for (size_t n = 0; n + 1 < f.size(); ++n) {
        if (f[n] < 0.0)
          throw std::runtime_error("read_tensor_csv: negative index on line " + std::to_string(ln));
        ix[n] = (uint64_t)f[n];
      }
      if (shape.empty()) shape.assign(ix.size(), 0);
      else if (shape.size() != ix.size())
        throw std::runtime_error("read_tensor_csv: inconsistent order on line " +
                                 std::to_string(ln));
      for (size_t n = 0; n < ix.size(); ++n) shape[n] = std::max(shape[n], ix[n] + 1);
      idx.push_back(std::move(ix));
      vals.push_back(f.back());
    }
    if (idx.empty()) throw std::runtime_error(std::string("read_tensor_csv: no entries in ") + path);
    const uint64_t vol = checked_volume(shape.data(), (uint32_t)shape.size());
    auto t = std::make_unique<rtucker_tensor>();
    t->shape = shape;
    t->host.assign(vol, 0.0);
    for (size_t k = 0; k < idx.size(); ++k) {
      uint64_t off = 0;
      for (size_t n = 0; n < shape.size(); ++n) off = off * shape[n] + idx[k][n];
      t->host[off] = vals[k];
    }
    check_finite(t->host.data(), vol, "DenseTensor");
    *out = t.release();
  });
}

rtucker_status rtucker_tensor_write(const rtucker_tensor* t, const char* path) {
  if (!t || !path) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    const double* hd = t->host_data();
    std::ofstream o(path, std::ios::binary | std::ios::trunc);
    if (!o) throw std::runtime_error(std::string("write_tensor: cannot open ") + path);
    o.write("DTEN", 4);
    wr<uint8_t>(o, 1);
    wr<uint32_t>(o, (uint32_t)t->shape.size());
    for (auto d : t->shape) wr<uint64_t>(o, d);
    o.write(reinterpret_cast<const char*>(hd), (std::streamsize)(t->size() * 8));
    if (!o) throw std::runtime_error(std::string("write_tensor: write failed for ") + path);
  });
}

uint32_t rtucker_tensor_order(const rtucker_tensor* t) {
  return t ? (uint32_t)t->shape.size() : 0;
}

rtucker_status rtucker_tensor_shape(const rtucker_tensor* t, uint64_t* shape_out) {
  if (!t || !shape_out) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  for (size_t n = 0; n < t->shape.size(); ++n) shape_out[n] = t->shape[n];
  return RTUCKER_OK;
}

uint64_t rtucker_tensor_size(const rtucker_tensor* t) { return t ? t->size() : 0; }

const double* rtucker_tensor_data(const rtucker_tensor* t) {
  if (!t) return nullptr;
  try {
    return t->host_data();
  } catch (const std::exception& e) {
    fail(RTUCKER_ERR_UNKNOWN, e.what());
    return nullptr;
  }
}

void rtucker_tensor_free(rtucker_tensor* t) { delete t; }

rtucker_status rtucker_tensor_generate(const uint64_t* shape, const uint64_t* planted_ranks,
                                       uint32_t order, double noise_fraction, double noise_sigma,
                                       uint64_t seed, rtucker_tensor** out,
                                       uint64_t* planted_checksum_out) {
  if (!shape || !planted_ranks || !out) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    // ref synthetic.cpp:31-70: uniform planted model, reconstruction (on the
    // GPU here), N(0, sigma) noise on round(fraction * size) distinct entries.
    if (noise_fraction < 0.0 || noise_fraction > 1.0)
      throw rtb::Error(1, "generate_synthetic: noise_fraction outside [0, 1]");
    const uint64_t total = checked_volume(shape, order);
    std::vector<uint64_t> sh(shape, shape + order), rk(planted_ranks, planted_ranks + order);
    uint64_t d = 1, fe = 0;
    for (uint32_t n = 0; n < order; ++n) {
      d *= rk[n];
    }
    Rng rng{seed};
    std::vector<double> core(d), fac;
    for (auto& v : core) v = rng.unit();
    for (uint32_t n = 0; n < order; ++n) {
      if (rk[n] == 0 || rk[n] > sh[n]) throw rtb::Error(1, "random_model: rank outside [1, I_n]");
      for (uint64_t i = 0; i < sh[n] * rk[n]; ++i) fac.push_back(rng.unit());
      fe += sh[n] * rk[n];
    }
    uint64_t h = 0xcbf29ce484222325ULL;
    const double lam = 0.0;
    h = fnv1a(&lam, 8, h);
    h = fnv1a(core.data(), d * 8, h);
    h = fnv1a(fac.data(), fe * 8, h);
    auto t = std::make_unique<rtucker_tensor>();
    t->shape = sh;
    t->host.resize(total);
    rtb::model_reconstruct(sh, rk, core.data(), fac.data(), t->host.data());
    const uint64_t count = (uint64_t)(noise_fraction * (double)total + 0.5);
    std::vector<uint64_t> chosen;
    chosen.reserve(count);
    if (count > 0) {
      if (count * 2 >= total) {
        std::vector<uint64_t> pool(total);
        for (uint64_t i = 0; i < total; ++i) pool[i] = i;
        for (uint64_t k = 0; k < count; ++k) {
          const uint64_t j = k + rng.below(total - k);
          std::swap(pool[k], pool[j]);
          chosen.push_back(pool[k]);
        }
      } else {
        std::unordered_set<uint64_t> seen;
        seen.reserve(count * 2);
        while (chosen.size() < count) {
          const uint64_t j = rng.below(total);
          if (seen.insert(j).second) chosen.push_back(j);
        }
      }
    }
    for (uint64_t j : chosen) t->host[j] += noise_sigma * rng.normal();
    if (planted_checksum_out) *planted_checksum_out = h;
    *out = t.release();
  });
}

void rtucker_als_options_init(rtucker_als_options* opts) {
  if (!opts) return;  // defaults of ref capi.cpp:163-174
  opts->lambda = 0.001;
  opts->sketched_core = 0;
  opts->epsilon = 0.1;
  opts->delta = 0.1;
  opts->seed = 0;
  opts->max_iterations = 50;
  opts->tolerance = 1e-6;
  opts->sample_count_override = 0;
  opts->record_history = 0;
}

// Multi-GPU: x holds this shard's rows of mode 1; the engine works on the global shape.
std::vector<uint64_t> engine_shape(const rtucker_tensor* x, const rtb::AlsOptions& o,
                                   const rtucker_b200_als_ext* ext) {
  std::vector<uint64_t> sh = x->shape;
  if (o.shard_count > 1) {
    if (!o.allreduce) throw rtb::Error(1, "sharded run needs an allreduce callback");
    const uint64_t total = ext->shard_rows_total;
    if (total == 0) throw rtb::Error(1, "sharded run needs shard_rows_total (global I_1)");
    if (o.shard_rank >= o.shard_count) throw rtb::Error(1, "shard_rank >= shard_count");
    const uint64_t lo = o.shard_rank * total / o.shard_count;
    const uint64_t hi = (o.shard_rank + 1) * total / o.shard_count;
    if (sh[0] != hi - lo)
      throw rtb::Error(1, "tensor rows != this shard's even split of shard_rows_total");
    sh[0] = total;
  }
  return sh;
}

static void apply_ext(rtb::AlsOptions& o, const rtucker_b200_als_ext* ext) {
  if (!ext) return;
  o.init_core = ext->init_core;
  o.init_factors = ext->init_factors;
  o.shard_rank = ext->shard_rank;
  o.shard_count = ext->shard_count ? ext->shard_count : 1;
  o.allreduce = ext->allreduce;
  o.allreduce_user = ext->allreduce_user;
  o.profile = ext->profile_kernels != 0;
  o.core_solver = ext->core_solver;
  o.fast_loss = ext->fast_loss != 0;
  o.factor_samples = ext->factor_samples;
  o.no_graph = ext->disable_graph != 0;
}

rtucker_status rtucker_b200_als_run_ex(const rtucker_tensor* x, const uint64_t* ranks,
                                       uint32_t order, const rtucker_als_options* opts,
                                       const rtucker_b200_als_ext* ext,
                                       rtucker_als_result** out) {
  if (!x || !ranks || !opts || !out) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    rtb::AlsOptions o = to_options(opts);
    if (order != x->shape.size()) throw rtb::Error(1, "als: ranks order != tensor order");
    if (o.max_iterations == 0) throw rtb::Error(1, "als: max_iterations must be >= 1");
    apply_ext(o, ext);
    auto r = std::make_unique<rtucker_als_result>();
    rtb::als_run(x->device(), engine_shape(x, o, ext), std::vector<uint64_t>(ranks, ranks + order),
                 o, r->out);
    *out = r.release();
  });
}

rtucker_status rtucker_als_run(const rtucker_tensor* x, const uint64_t* ranks, uint32_t order,
                               const rtucker_als_options* opts, rtucker_als_result** out) {
  return rtucker_b200_als_run_ex(x, ranks, order, opts, nullptr, out);
}

struct rtucker_b200_session {
  std::unique_ptr<rtb::Session> s;
  std::vector<double> init_core, init_factors;
};

rtucker_status rtucker_b200_session_create(const rtucker_tensor* x, const uint64_t* ranks,
                                           uint32_t order, const rtucker_als_options* opts,
                                           const rtucker_b200_als_ext* ext,
                                           rtucker_b200_session** out) {
  if (!x || !ranks || !opts || !out) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    rtb::AlsOptions o = to_options(opts);
    if (order != x->shape.size()) throw rtb::Error(1, "als: ranks order != tensor order");
    apply_ext(o, ext);
    auto s = std::make_unique<rtucker_b200_session>();
    s->s.reset(rtb::session_create(x->device(), engine_shape(x, o, ext),
                                   std::vector<uint64_t>(ranks, ranks + order), o));
    *out = s.release();
  });
}

rtucker_status rtucker_b200_session_sweeps(rtucker_b200_session* s, uint32_t n) {
  if (!s) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] { rtb::session_run(s->s.get(), n, false); });
}

rtucker_status rtucker_b200_session_result(rtucker_b200_session* s, rtucker_als_result** out) {
  if (!s || !out) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    auto r = std::make_unique<rtucker_als_result>();
    rtb::session_output(s->s.get(), r->out);
    *out = r.release();
  });
}

void rtucker_b200_session_free(rtucker_b200_session* s) { delete s; }

uint64_t rtucker_result_history_size(const rtucker_als_result* r) {
  return r ? r->out.history.size() : 0;
}

rtucker_status rtucker_result_history_row(const rtucker_als_result* r, uint64_t i,
                                          uint32_t* iteration, char* step_buf, size_t step_buf_len,
                                          double* loss, double* rmse) {
  if (!r || i >= r->out.history.size())
    return fail(RTUCKER_ERR_INVALID_ARGUMENT, "history row out of range");
  const auto& row = r->out.history[i];
  if (iteration) *iteration = row.iteration;
  if (loss) *loss = row.loss;
  if (rmse) *rmse = row.rmse;
  return copy_label(row.step, step_buf, step_buf_len);
}

uint64_t rtucker_result_timing_size(const rtucker_als_result* r) {
  return r ? r->out.timings.size() : 0;
}

rtucker_status rtucker_result_timing_row(const rtucker_als_result* r, uint64_t i, char* step_buf,
                                         size_t step_buf_len, double* mean_seconds,
                                         uint64_t* count) {
  if (!r || i >= r->out.timings.size())
    return fail(RTUCKER_ERR_INVALID_ARGUMENT, "timing row out of range");
  const auto& t = r->out.timings[i];
  if (mean_seconds) *mean_seconds = t.count ? t.total / (double)t.count : 0.0;
  if (count) *count = t.count;
  return copy_label(t.step, step_buf, step_buf_len);
}

double rtucker_result_final_loss(const rtucker_als_result* r) { return r ? r->out.final_loss : 0.0; }
double rtucker_result_final_rmse(const rtucker_als_result* r) { return r ? r->out.final_rmse : 0.0; }
uint32_t rtucker_result_iterations(const rtucker_als_result* r) {
  return r ? r->out.iterations : 0;
}

rtucker_status rtucker_result_model(const rtucker_als_result* r, rtucker_model** out) {
  if (!r || !out) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] { *out = model_from_output(r->out); });
}

void rtucker_result_free(rtucker_als_result* r) { delete r; }

rtucker_status rtucker_model_write(const rtucker_model* m, const char* path) {
  if (!m || !path) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    // RTKM1 (ref model_io.cpp:29-52)
    std::ofstream o(path, std::ios::binary | std::ios::trunc);
    if (!o) throw std::runtime_error(std::string("write_model: cannot open ") + path);
    o.write("RTKM", 4);
    wr<uint8_t>(o, 1);
    wr<double>(o, m->lambda);
    wr<uint32_t>(o, (uint32_t)m->ranks.size());
    for (auto r : m->ranks) wr<uint64_t>(o, r);
    o.write(reinterpret_cast<const char*>(m->core.data()), (std::streamsize)(m->core.size() * 8));
    uint64_t off = 0;
    for (size_t n = 0; n < m->ranks.size(); ++n) {
      wr<uint64_t>(o, m->shape[n]);
      wr<uint64_t>(o, m->ranks[n]);
      o.write(reinterpret_cast<const char*>(m->factors.data() + off),
              (std::streamsize)(m->shape[n] * m->ranks[n] * 8));
      off += m->shape[n] * m->ranks[n];
    }
    if (!o) throw std::runtime_error(std::string("write_model: write failed for ") + path);
  });
}

rtucker_status rtucker_model_read(const char* path, rtucker_model** out) {
  if (!path || !out) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    // RTKM1 (ref model_io.cpp:54-99)
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error(std::string("read_model: cannot open ") + path);
    char magic[4];
    in.read(magic, 4);
    if (!in || std::memcmp(magic, "RTKM", 4) != 0)
      throw std::runtime_error(std::string("read_model: bad magic in ") + path);
    if (rd<uint8_t>(in, "read_model: truncated version") != 1)
      throw std::runtime_error("read_model: unsupported version");
    auto m = std::make_unique<rtucker_model>();
    m->lambda = rd<double>(in, "read_model: truncated lambda");
    const uint32_t order = rd<uint32_t>(in, "read_model: truncated order");
    if (order == 0 || order > 8) throw std::runtime_error("read_model: order outside [1, 8]");
    uint64_t cs = 1;
    for (uint32_t n = 0; n < order; ++n) {
      m->ranks.push_back(rd<uint64_t>(in, "read_model: truncated core shape"));
      cs *= m->ranks.back();
    }
    m->core.resize(cs);
    in.read(reinterpret_cast<char*>(m->core.data()), (std::streamsize)(cs * 8));
    if (!in) throw std::runtime_error("read_model: truncated core payload");
    for (uint32_t n = 0; n < order; ++n) {
      const uint64_t rows = rd<uint64_t>(in, "read_model: truncated factor rows");
      const uint64_t cols = rd<uint64_t>(in, "read_model: truncated factor cols");
      m->shape.push_back(rows);
      if (cols != m->ranks[n]) throw rtb::Error(1, "read_model: factor/core shape mismatch");
      const size_t off = m->factors.size();
      m->factors.resize(off + rows * cols);
      in.read(reinterpret_cast<char*>(m->factors.data() + off), (std::streamsize)(rows * cols * 8));
      if (!in) throw std::runtime_error("read_model: truncated factor payload");
    }
    check_finite(m->core.data(), m->core.size(), "DenseTensor");
    check_finite(m->factors.data(), m->factors.size(), "DenseMatrix");
    *out = m.release();
  });
}

rtucker_status rtucker_model_reconstruct(const rtucker_model* m, rtucker_tensor** out) {
  if (!m || !out) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    auto t = std::make_unique<rtucker_tensor>();
    t->shape = m->shape;
    t->host.resize(t->size());
    rtb::model_reconstruct(m->shape, m->ranks, m->core.data(), m->factors.data(), t->host.data());
    *out = t.release();
  });
}

double rtucker_model_lambda(const rtucker_model* m) { return m ? m->lambda : 0.0; }
uint32_t rtucker_model_order(const rtucker_model* m) { return m ? (uint32_t)m->ranks.size() : 0; }
rtucker_status rtucker_model_ranks(const rtucker_model* m, uint64_t* ranks_out) {
  if (!m || !ranks_out) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  for (size_t n = 0; n < m->ranks.size(); ++n) ranks_out[n] = m->ranks[n];
  return RTUCKER_OK;
}
void rtucker_model_free(rtucker_model* m) { delete m; }

rtucker_status rtucker_solve_ridge(const double* a, uint64_t n, uint64_t d, const double* b,
                                   double lambda, double* x_out) {
  if (!a || !b || !x_out) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    check_finite(a, n * d, "DenseMatrix");
    rtb::dense_solve_ridge(a, n, d, b, lambda, x_out);
  });
}

rtucker_status rtucker_ridge_scores(const double* a, uint64_t n, uint64_t d, double lambda,
                                    double* scores_out) {
  if (!a || !scores_out) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    check_finite(a, n * d, "DenseMatrix");
    rtb::dense_ridge_scores(a, n, d, lambda, scores_out);
  });
}

rtucker_status rtucker_sketched_ridge(const double* a, uint64_t n, uint64_t d, const double* b,
                                      const double* candidate_scores, double lambda,
                                      double d_eff_lower, double epsilon, double delta,
                                      uint64_t sample_count_override, uint64_t seed, double* x_out,
                                      uint64_t* sample_count_out, double* beta_prime_out) {
  if (!a || !b || !x_out) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    check_finite(a, n * d, "DenseMatrix");
    rtb::dense_sketched_ridge(a, n, d, b, candidate_scores, lambda, d_eff_lower, epsilon, delta,
                              sample_count_override, seed, x_out, sample_count_out,
                              beta_prime_out);
  });
}

rtucker_status rtucker_verify_suite(const char* name, uint64_t seed, int* passed_out,
                                    char** json_report_out) {
  if (!name || !passed_out) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    // ref capi.cpp:364-403; the suites run against the GPU routines (verify.cu)
    std::string json;
    const bool ok = rtb::verify_suites(name, seed, json);
    *passed_out = ok ? 1 : 0;
    if (json_report_out) {
      char* buf = new char[json.size() + 1];
      std::memcpy(buf, json.c_str(), json.size() + 1);
      *json_report_out = buf;
    }
  });
}

void rtucker_string_free(char* s) { delete[] s; }

// ---- extensions (rtucker_b200.h) ----

rtucker_status rtucker_b200_set_device(int device) {
  return guarded([&] { RTB_CUDA(cudaSetDevice(device)); });
}

unsigned long long rtucker_b200_launch_count(void) { return rtb::launch_counter(); }

uint64_t rtucker_b200_result_graph_sweeps(const rtucker_als_result* r) {
  return r ? r->out.graph_launches : 0;
}

unsigned long long rtucker_b200_variant_count(const char* name) {
  return name ? rtb::variant_count(name) : 0;
}

rtucker_status rtucker_b200_set_stream(void* stream) {
  rtb::set_stream(static_cast<cudaStream_t>(stream));
  return RTUCKER_OK;
}

rtucker_status rtucker_b200_tensor_create_device(const uint64_t* shape, uint32_t order,
                                                 const double* data_device, rtucker_tensor** out) {
  if (!shape || !data_device || !out) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    const uint64_t v = checked_volume(shape, order);
    auto t = std::make_unique<rtucker_tensor>();
    t->shape.assign(shape, shape + order);
    t->host_valid = false;
    cudaStream_t st = rtb::current_stream();
    t->dev.ensure(v * 8, st);
    RTB_CUDA(cudaMemcpyAsync(t->dev.p, data_device, v * 8, cudaMemcpyDeviceToDevice, st));
    // the caller may free or reuse the source as soon as we return
    RTB_CUDA(cudaStreamSynchronize(st));
    t->dev_valid = true;
    *out = t.release();
  });
}

rtucker_status rtucker_b200_tensor_generate_device(const uint64_t* shape,
                                                   const uint64_t* planted_ranks, uint32_t order,
                                                   double noise_level, double pareto_alpha,
                                                   uint64_t seed, uint32_t shard_rank,
                                                   uint32_t shard_count, rtucker_tensor** out,
                                                   double* core_out, double* factors_out) {
  if (!shape || !planted_ranks || !out) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    checked_volume(shape, order);
    const uint32_t P = shard_count ? shard_count : 1;
    if (shard_rank >= P || P > shape[0]) throw rtb::Error(1, "generate: bad shard");
    std::vector<uint64_t> sh(shape, shape + order), rk(planted_ranks, planted_ranks + order);
    auto t = std::make_unique<rtucker_tensor>();
    t->shape = sh;
    t->shape[0] = (uint64_t)(shard_rank + 1) * shape[0] / P - (uint64_t)shard_rank * shape[0] / P;
    t->host_valid = false;
    cudaStream_t st = rtb::current_stream();
    t->dev.ensure(t->size() * 8, st);
    rtb::generate_planted_device(sh, rk, noise_level, pareto_alpha, seed, shard_rank, P,
                                 t->dev.as<double>(), core_out, factors_out);
    t->dev_valid = true;
    *out = t.release();
  });
}

const double* rtucker_b200_tensor_device_data(const rtucker_tensor* t) {
  if (!t) return nullptr;
  try {
    return t->device();
  } catch (const std::exception& e) {
    fail(RTUCKER_ERR_UNKNOWN, e.what());
    return nullptr;
  }
}

rtucker_status rtucker_b200_model_data(const rtucker_model* m, double* core_out,
                                       double* factors_out) {
  if (!m) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  if (core_out) std::memcpy(core_out, m->core.data(), m->core.size() * 8);
  if (factors_out) std::memcpy(factors_out, m->factors.data(), m->factors.size() * 8);
  return RTUCKER_OK;
}

rtucker_status rtucker_b200_model_create(const uint64_t* shape, const uint64_t* ranks,
                                         uint32_t order, const double* core,
                                         const double* factors, double lambda,
                                         rtucker_model** out) {
  if (!shape || !ranks || !core || !factors || !out)
    return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    checked_volume(shape, order);
    auto m = std::make_unique<rtucker_model>();
    m->shape.assign(shape, shape + order);
    m->ranks.assign(ranks, ranks + order);
    uint64_t d = 1, fe = 0;
    for (uint32_t n = 0; n < order; ++n) {
      if (ranks[n] == 0) throw rtb::Error(1, "DenseTensor: zero-length dimension");
      d *= ranks[n];
      fe += shape[n] * ranks[n];
    }
    m->core.assign(core, core + d);
    m->factors.assign(factors, factors + fe);
    check_finite(m->core.data(), d, "DenseTensor");
    check_finite(m->factors.data(), fe, "DenseMatrix");
    m->lambda = lambda;
    *out = m.release();
  });
}

rtucker_status rtucker_b200_result_sketch_info(const rtucker_als_result* r, uint64_t* sample_count,
                                               uint64_t* data_draws, int* rank_deficient,
                                               int* solver_path) {
  if (!r) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  if (sample_count) *sample_count = r->out.last_sample_count;
  if (data_draws) *data_draws = r->out.last_data_draws;
  if (rank_deficient) *rank_deficient = r->out.last_rank_deficient;
  if (solver_path) *solver_path = r->out.last_solver_path;
  return RTUCKER_OK;
}

int rtucker_b200_result_pcg_iterations(const rtucker_als_result* r) {
  return r ? r->out.last_pcg_iterations : 0;
}

uint64_t rtucker_b200_result_kernel_count(const rtucker_als_result* r) {
  return r ? r->out.kernels.size() : 0;
}

rtucker_status rtucker_b200_result_kernel_row(const rtucker_als_result* r, uint64_t i,
                                              char* name_buf, size_t name_len,
                                              double* total_seconds, uint64_t* launches) {
  if (!r || i >= r->out.kernels.size())
    return fail(RTUCKER_ERR_INVALID_ARGUMENT, "kernel row out of range");
  const auto& k = r->out.kernels[i];
  if (total_seconds) *total_seconds = k.total;
  if (launches) *launches = k.launches;
  return copy_label(k.name, name_buf, name_len);
}

double rtucker_b200_result_sweep_seconds(const rtucker_als_result* r) {
  return r ? r->out.sweep_seconds : 0.0;
}

rtucker_status rtucker_b200_factor_scores(const double* factor, uint64_t rows, uint64_t cols,
                                          double* scores_out, double* cdf_out, double* sum_out,
                                          uint64_t* rank_out) {
  if (!factor || !scores_out || !cdf_out || !sum_out)
    return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    check_finite(factor, rows * cols, "DenseMatrix");
    uint64_t rk = 0;
    rtb::factor_scores(factor, (int)rows, (int)cols, scores_out, cdf_out, sum_out, &rk);
    if (rank_out) *rank_out = rk;
  });
}

rtucker_status rtucker_b200_kron_draw(uint32_t order, const uint64_t* rows, uint64_t d,
                                      const double* scores, const double* cdfs,
                                      const double* sums, uint64_t seed, uint64_t s,
                                      uint64_t* indices_out, double* weights_out) {
  if (!rows || !scores || !cdfs || !sums || !indices_out || !weights_out)
    return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    rtb::kron_draw((int)order, rows, d, scores, cdfs, sums, seed, s, indices_out, weights_out);
  });
}

rtucker_status rtucker_b200_kron_fiber_sketch_shard(
    const float* x_dev, const uint64_t* shape, uint32_t x_layout, const double* a2_dev,
    const double* a3_dev, uint32_t r2, uint32_t r3, double lambda, uint64_t s, uint64_t seed,
    double* gram_dev, double* rhs_dev, uint64_t* indices_out, double* weights_out,
    uint64_t* data_draws_out, uint64_t* unique_rows_out, double* phase_ms_out,
    uint32_t shard_rank, uint32_t shard_count) {
  return guarded([&] {
    if (!shape || !a2_dev || !a3_dev) throw rtb::Error(1, "kron_fiber_sketch: null argument");
    if (x_layout > 1) throw rtb::Error(1, "kron_fiber_sketch: x_layout must be 0 or 1");
    if (shard_count < 1 || shard_rank >= shard_count)
      throw rtb::Error(1, "kron_fiber_sketch: bad shard");
    rtb::kron_fiber_sketch(x_dev, x_layout == 1, (int)shape[0], (int)shape[1], (int)shape[2],
                           a2_dev, a3_dev, (int)r2, (int)r3, lambda, s, seed, gram_dev, rhs_dev,
                           indices_out, weights_out, data_draws_out, unique_rows_out,
                           phase_ms_out, (int)shard_rank, (int)shard_count);
  });
}

rtucker_status rtucker_b200_kron_fiber_sketch(const float* x_dev, const uint64_t* shape,
                                              uint32_t x_layout, const double* a2_dev,
                                              const double* a3_dev, uint32_t r2, uint32_t r3,
                                              double lambda, uint64_t s, uint64_t seed,
                                              double* gram_dev, double* rhs_dev,
                                              uint64_t* indices_out, double* weights_out,
                                              uint64_t* data_draws_out, uint64_t* unique_rows_out,
                                              double* phase_ms_out) {
  return rtucker_b200_kron_fiber_sketch_shard(x_dev, shape, x_layout, a2_dev, a3_dev, r2, r3,
                                              lambda, s, seed, gram_dev, rhs_dev, indices_out,
                                              weights_out, data_draws_out, unique_rows_out,
                                              phase_ms_out, 0, 1);
}

rtucker_status rtucker_b200_tensor_fiber_major(const float* x_dev, const uint64_t* shape,
                                               float* out_dev) {
  return guarded([&] {
    if (!x_dev || !shape || !out_dev) throw rtb::Error(1, "tensor_fiber_major: null argument");
    if (shape[0] < 1 || shape[1] < 1 || shape[2] < 1 || shape[0] > 0x7fffffffULL ||
        shape[1] > 0x7fffffffULL || shape[2] > 0x7fffffffULL)
      throw rtb::Error(1, "tensor_fiber_major: bad shape");
    rtb::tensor_fiber_major(x_dev, (int)shape[0], (int)shape[1], (int)shape[2], out_dev);
  });
}

rtucker_status rtucker_b200_kron_normal_eq(uint32_t order, const uint64_t* rows,
                                           const uint64_t* ranks, const double* factors,
                                           const double* x, double lambda, uint64_t s,
                                           const uint64_t* indices, const double* weights,
                                           double* gram_out, double* rhs_out) {
  if (!rows || !ranks || !factors || !x || !indices || !weights || !gram_out || !rhs_out)
    return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    rtb::kron_normal_eq((int)order, rows, ranks, factors, x, lambda, s, indices, weights, gram_out,
                        rhs_out);
  });
}

rtucker_status rtucker_b200_aug_draw(const double* candidate_scores, uint64_t n, uint64_t d,
                                     double d_eff_lower, uint64_t seed, uint64_t s,
                                     uint64_t* indices_out, double* weights_out) {
  if (!candidate_scores || !indices_out || !weights_out)
    return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded(
      [&] { rtb::aug_draw(candidate_scores, n, d, d_eff_lower, seed, s, indices_out, weights_out); });
}

rtucker_status rtucker_b200_dense_normal_eq(const double* a, uint64_t n, uint64_t d,
                                            const double* b, double lambda, uint64_t s,
                                            const uint64_t* indices, const double* weights,
                                            double* gram_out, double* rhs_out) {
  if (!a || !b || !indices || !weights || !gram_out || !rhs_out)
    return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded(
      [&] { rtb::dense_normal_eq(a, n, d, b, lambda, s, indices, weights, gram_out, rhs_out); });
}

rtucker_status rtucker_b200_sample_count(double beta_prime, uint64_t d, double epsilon,
                                         double delta, uint64_t* out) {
  if (!out) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] { *out = rtb::sample_count_formula(beta_prime, d, epsilon, delta); });
}

rtucker_status rtucker_b200_sym_eig(const double* a, uint64_t d, double* evals_out,
                                    double* evecs_out) {
  if (!a || !evals_out || !evecs_out) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] { rtb::sym_eig(a, d, evals_out, evecs_out); });
}

rtucker_status rtucker_b200_spd_solve(const double* gram, const double* rhs, uint64_t d,
                                      double* x_out, uint64_t* rank_out, int* path_out) {
  if (!gram || !rhs || !x_out) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] { rtb::spd_solve(gram, rhs, d, x_out, rank_out, path_out); });
}

rtucker_status rtucker_b200_update_core_sketched(const rtucker_tensor* x, const rtucker_model* m,
                                                 uint64_t s, uint64_t seed, double* core_out,
                                                 uint64_t* indices_out, double* weights_out) {
  if (!x || !m || !core_out) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    if (x->shape != m->shape) throw rtb::Error(1, "tucker: factor/core/tensor shape mismatch");
    rtb::model_update_core_sketched(x->device(), m->shape, m->ranks, m->core.data(),
                                    m->factors.data(), m->lambda, s, seed, core_out, indices_out,
                                    weights_out);
  });
}

rtucker_status rtucker_b200_update_factor(const rtucker_tensor* x, const rtucker_model* m,
                                          uint32_t mode, double* factor_out) {
  if (!x || !m || !factor_out) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    if (x->shape != m->shape) throw rtb::Error(1, "tucker: factor/core/tensor shape mismatch");
    rtb::model_update_factor(x->device(), m->shape, m->ranks, m->core.data(), m->factors.data(),
                             m->lambda, mode, factor_out);
  });
}

rtucker_status rtucker_b200_update_core_exact(const rtucker_tensor* x, const rtucker_model* m,
                                              double* core_out) {
  if (!x || !m || !core_out) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    if (x->shape != m->shape) throw rtb::Error(1, "tucker: factor/core/tensor shape mismatch");
    rtb::model_update_core_exact(x->device(), m->shape, m->ranks, m->core.data(),
                                 m->factors.data(), m->lambda, core_out);
  });
}

rtucker_status rtucker_b200_loss(const rtucker_tensor* x, const rtucker_model* m,
                                 double* loss_out, double* rmse_out) {
  if (!x || !m || !loss_out) return fail(RTUCKER_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    if (x->shape != m->shape) throw rtb::Error(1, "tucker: factor/core/tensor shape mismatch");
    double rm = 0.0;
    rtb::model_loss(x->device(), m->shape, m->ranks, m->core.data(), m->factors.data(), m->lambda,
                    loss_out, &rm);
    if (rmse_out) *rmse_out = rm;
  });
}

}  // extern "C"
