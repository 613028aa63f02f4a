// tt_engine.hpp -- header-only C++ wrapper over the C-ABI (tt_engine.h) with
// the reference's call shapes and exception types (namespace ttgnn,
// proj/core/include/ttgnn/{tt_embedding,autodiff}.hpp):
//
//   DeviceTT::lookup_batch     lookup_batch     tt_embedding.hpp:55 / .cpp:110-125
//   DeviceTT::backward_lookup  backward_lookup  autodiff.hpp:39-41 / .cpp:48-118
//   DeviceTT::make_optimizer   OptimizerState::make  autodiff.hpp:55 / .cpp:120-133 (+ Adagrad)
//   DeviceTT::apply_update     apply_update     autodiff.hpp:60 / .cpp:147-173
//
// Errors are rethrown as the reference throws them: std::out_of_range for an
// index outside [0, num_nodes) (with the first offending batch position),
// std::invalid_argument for shape mismatches and non-finite gradients (with
// cores, moments and step untouched), std::runtime_error otherwise.
//
// A ttgnn maintainer's shim converts TTEmbedding / MatrixRM
// to and from the plain vectors used here; tests/cpp/shim_test.cpp drives this
// header against the oracle from pytest.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "tt_engine.h"

namespace tt_b200 {

enum class OptKind { sgd = TT_OPT_SGD, adam = TT_OPT_ADAM, adagrad = TT_OPT_ADAGRAD };

struct IndexError : std::out_of_range {
  int64_t position, value;
  IndexError(const std::string& m, int64_t p, int64_t v) : std::out_of_range(m), position(p), value(v) {}
};

inline void check(int rc) {
  if (rc == TT_OK) return;
  const std::string msg = tt_last_error();
  if (rc == TT_ERR_INDEX) throw IndexError(msg, tt_last_error_position(), tt_last_error_value());
  if (rc == TT_ERR_ARG || rc == TT_ERR_NONFINITE) throw std::invalid_argument(msg);
  if (rc == TT_ERR_NOMEM) throw std::bad_alloc();
  throw std::runtime_error(msg);
}

struct Config {  // TTConfig (tt_config.hpp:33-52)
  int64_t num_nodes = 0, emb_dim = 0;
  std::vector<int64_t> row_factors, col_factors, ranks;

  tt_config_c c_abi() const {
    tt_config_c c{};
    c.num_nodes = num_nodes;
    c.emb_dim = emb_dim;
    c.d = (int32_t)row_factors.size();
    if (c.d > TT_MAX_CORES || col_factors.size() != row_factors.size() || ranks.size() != row_factors.size() + 1)
      throw std::invalid_argument("TTConfig: factor / rank counts inconsistent");
    for (int k = 0; k < c.d; ++k) {
      c.row_factors[k] = row_factors[k];
      c.col_factors[k] = col_factors[k];
    }
    for (int k = 0; k <= c.d; ++k) c.ranks[k] = ranks[k];
    return c;
  }
  int d() const { return (int)row_factors.size(); }
  int64_t core_size(int k) const { return ranks[k] * row_factors[k] * col_factors[k] * ranks[k + 1]; }
};

// One handle per GPU: device cores, gradients, optimizer state, plan scratch.
class DeviceTT {
 public:
  DeviceTT(const Config& cfg, int device = 0) : cfg_(cfg) {
    const tt_config_c c = cfg.c_abi();
    check(tt_config_validate(&c));
    check(tt_engine_create(&c, device, &h_));
  }
  ~DeviceTT() { tt_engine_destroy(h_); }
  DeviceTT(const DeviceTT&) = delete;
  DeviceTT& operator=(const DeviceTT&) = delete;

  tt_engine* handle() const { return h_; }
  const Config& config() const { return cfg_; }

  // cores in the reference layout (R_{k-1}, m_k, n_k, R_k), row-major
  void set_cores(const std::vector<std::vector<double>>& cores) {
    if ((int)cores.size() != cfg_.d()) throw std::invalid_argument("TTEmbedding: wrong number of cores");
    std::vector<const double*> p;
    for (int k = 0; k < cfg_.d(); ++k) {
      if ((int64_t)cores[k].size() != cfg_.core_size(k))
        throw std::invalid_argument("TTEmbedding: core " + std::to_string(k) + " storage size mismatch");
      p.push_back(cores[k].data());
    }
    check(tt_set_cores_f64(h_, p.data()));
  }
  std::vector<std::vector<double>> cores() const {
    std::vector<std::vector<double>> out(cfg_.d());
    std::vector<double*> p;
    for (int k = 0; k < cfg_.d(); ++k) {
      out[k].resize((size_t)cfg_.core_size(k));
      p.push_back(out[k].data());
    }
    check(tt_get_cores_f64(h_, p.data()));
    return out;
  }

  // lookup_batch: B x emb_dim row-major
  std::vector<float> lookup_batch(const std::vector<int64_t>& idx) const {
    std::vector<float> out(idx.size() * (size_t)cfg_.emb_dim);
    check(tt_lookup_batch(h_, idx.data(), (int64_t)idx.size(), out.data()));
    return out;
  }

  // backward_lookup: gradients stay on the device; CoreGradients on demand
  void backward_lookup(const std::vector<int64_t>& idx, const std::vector<float>& upstream) {
    if (upstream.size() != idx.size() * (size_t)cfg_.emb_dim)
      throw std::invalid_argument("backward_lookup: upstream shape mismatch");
    check(tt_backward_lookup(h_, idx.data(), (int64_t)idx.size(), upstream.data()));
  }
  std::vector<std::vector<double>> core_grads(int64_t* batch_count = nullptr) const {
    std::vector<std::vector<double>> out(cfg_.d());
    std::vector<double*> p;
    for (int k = 0; k < cfg_.d(); ++k) {
      out[k].resize((size_t)cfg_.core_size(k));
      p.push_back(out[k].data());
    }
    check(tt_get_core_grads_f64(h_, p.data(), batch_count));
    return out;
  }
  void set_core_grads(const std::vector<std::vector<double>>& g, int64_t batch_count) {
    std::vector<const double*> p;
    for (auto& x : g) p.push_back(x.data());
    check(tt_set_core_grads_f64(h_, p.data(), batch_count));
  }

  // OptimizerState::make (+ Adagrad): eps defaults 1e-8 (Adam), 1e-10 (Adagrad)
  void make_optimizer(OptKind k, double lr) { check(tt_opt_init(h_, (int)k, lr, 0, 0, 0)); }
  void set_learning_rate(double lr) { check(tt_opt_set_hparams(h_, lr, 0, 0, 0)); }
  int64_t step() const {
    int64_t s = 0;
    check(tt_opt_get_step(h_, &s));
    return s;
  }
  // apply_update: all-or-nothing
  void apply_update() { check(tt_apply_update(h_)); }

  // device-buffer hot path (stream-ordered; errors deferred to sync())
  void forward(const int64_t* d_idx, int64_t B, float* d_out, void* stream) { check(tt_forward(h_, d_idx, B, d_out, stream)); }
  void backward(const int64_t* d_idx, int64_t B, const float* d_up, void* stream) {
    check(tt_backward(h_, d_idx, B, d_up, stream));
  }
  void update(void* stream) { check(tt_step(h_, stream)); }
  void sync(void* stream) { check(tt_sync(h_, stream)); }

  // one step through host memory (indices / upstream up, rows down)
  void train_step_host(const std::vector<int64_t>& idx, const std::vector<float>& up, std::vector<float>* rows) {
    if (rows) rows->resize(idx.size() * (size_t)cfg_.emb_dim);
    check(tt_train_step_host(h_, idx.data(), (int64_t)idx.size(), up.data(), rows ? rows->data() : nullptr));
  }

  // NCCL position sharding
  static std::vector<char> nccl_unique_id() {
    std::vector<char> id(128);
    check(tt_nccl_unique_id(id.data(), (int64_t)id.size()));
    return id;
  }
  void comm_init_rank(const std::vector<char>& id, int rank, int nranks) {
    check(tt_comm_init_rank(h_, id.data(), rank, nranks));
  }
  void allreduce_grads(void* stream) { check(tt_allreduce_grads(h_, stream)); }

  // NCCL ID-owner sharding (device buffers, stream-ordered)
  void owner_forward(const int64_t* d_idx, int64_t B, float* d_out, void* stream) {
    check(tt_owner_forward(h_, d_idx, B, d_out, stream));
  }
  void owner_backward(const float* d_up, void* stream) { check(tt_owner_backward(h_, d_up, stream)); }
  void owner_step(void* stream) { check(tt_owner_step(h_, stream)); }

 private:
  Config cfg_;
  tt_engine* h_ = nullptr;
};

}  // namespace tt_b200
