// shim_test.cpp -- a C++ host driving the engine through include/tt_engine.hpp
// (the C-ABI with the reference's call shapes and exception types), as the
// reference's own C++ training loop would (gnn.cpp:89-128, 313-411).
//
// Usage: shim_test <dir>
//   <dir>/cfg.txt           num_nodes emb_dim d / m... / n... / R...
//   <dir>/core<k>.f64       cores, reference layout (R, m, n, R)
//   <dir>/idx.i64           B indices;  <dir>/up.f32  B x emb_dim upstream
// Writes (compared with the oracle by tests/test_cpp_shim.py):
//   rows.f32                lookup_batch
//   grad<k>.f64             backward_lookup -> CoreGradients
//   adagrad<k>.f64          cores after OptimizerState::make(adagrad, 0.01) + apply_update
//   comm<k>.f64             cores after the same step on an engine with a 1-rank NCCL
//                           communicator (device path + tt_allreduce_grads)
// and checks the error contract itself (exit code != 0 on a failed check).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "tt_engine.hpp"

using tt_b200::Config;
using tt_b200::DeviceTT;
using tt_b200::OptKind;

static int failures = 0;
#define CHECK(cond, what)                                               \
  do {                                                                  \
    if (!(cond)) {                                                      \
      std::cerr << "FAILED: " << what << " (" #cond ")\n";              \
      ++failures;                                                       \
    }                                                                   \
  } while (0)

template <class T>
std::vector<T> read_raw(const std::string& path) {
  std::ifstream f(path, std::ios::binary | std::ios::ate);
  if (!f) throw std::runtime_error("cannot open " + path);
  const std::streamsize n = f.tellg();
  f.seekg(0);
  std::vector<T> v((size_t)n / sizeof(T));
  f.read(reinterpret_cast<char*>(v.data()), n);
  return v;
}

template <class T>
void write_raw(const std::string& path, const std::vector<T>& v) {
  std::ofstream f(path, std::ios::binary);
  f.write(reinterpret_cast<const char*>(v.data()), (std::streamsize)(v.size() * sizeof(T)));
}

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: shim_test <dir>\n";
    return 2;
  }
  const std::string dir = argv[1];
  Config cfg;
  {
    std::ifstream f(dir + "/cfg.txt");
    int d = 0;
    f >> cfg.num_nodes >> cfg.emb_dim >> d;
    cfg.row_factors.resize(d);
    cfg.col_factors.resize(d);
    cfg.ranks.resize(d + 1);
    for (auto& x : cfg.row_factors) f >> x;
    for (auto& x : cfg.col_factors) f >> x;
    for (auto& x : cfg.ranks) f >> x;
  }
  const int d = cfg.d();
  std::vector<std::vector<double>> cores(d);
  for (int k = 0; k < d; ++k) cores[k] = read_raw<double>(dir + "/core" + std::to_string(k) + ".f64");
  const std::vector<int64_t> idx = read_raw<int64_t>(dir + "/idx.i64");
  const std::vector<float> up = read_raw<float>(dir + "/up.f32");
  const int64_t B = (int64_t)idx.size();

  try {
    // ---- the reference call sequence, host buffers ----------------------
    DeviceTT emb(cfg, 0);
    emb.set_cores(cores);
    write_raw(dir + "/rows.f32", emb.lookup_batch(idx));
    emb.backward_lookup(idx, up);
    int64_t bc = -1;
    const auto g = emb.core_grads(&bc);
    CHECK(bc == B, "CoreGradients::batch_count");
    for (int k = 0; k < d; ++k) write_raw(dir + "/grad" + std::to_string(k) + ".f64", g[k]);
    emb.make_optimizer(OptKind::adagrad, 0.01);
    emb.apply_update();
    CHECK(emb.step() == 1, "step after one apply_update");
    const auto after = emb.cores();
    for (int k = 0; k < d; ++k) write_raw(dir + "/adagrad" + std::to_string(k) + ".f64", after[k]);

    // ---- error contract (tt_embedding.cpp:112-117, autodiff.cpp:53-60, :155-158)
    {
      std::vector<int64_t> bad = {0, 1, cfg.num_nodes, -1};
      bool threw = false;
      try {
        emb.lookup_batch(bad);
      } catch (const tt_b200::IndexError& e) {
        threw = true;
        CHECK(e.position == 2 && e.value == cfg.num_nodes, "out_of_range names the first bad position");
        CHECK(std::string(e.what()).find("position 2") != std::string::npos, "message names the position");
      }
      CHECK(threw, "lookup_batch throws std::out_of_range");
      threw = false;
      try {
        emb.backward_lookup({0, 1}, std::vector<float>(3 * cfg.emb_dim));
      } catch (const std::invalid_argument&) {
        threw = true;
      }
      CHECK(threw, "backward_lookup shape mismatch throws std::invalid_argument");
      // non-finite gradient: rejected, cores and step untouched
      auto ng = g;
      ng[d - 1][0] = std::nan("");
      emb.set_core_grads(ng, B);
      threw = false;
      try {
        emb.apply_update();
      } catch (const std::invalid_argument& e) {
        threw = true;
        CHECK(std::string(e.what()).find("core " + std::to_string(d - 1)) != std::string::npos, "names the core");
      }
      CHECK(threw, "non-finite gradient throws std::invalid_argument");
      CHECK(emb.step() == 1, "rejected update leaves the step");
      const auto same = emb.cores();
      bool eq = true;
      for (int k = 0; k < d; ++k) eq = eq && std::memcmp(same[k].data(), after[k].data(), after[k].size() * 8) == 0;
      CHECK(eq, "rejected update leaves the cores");
      // the engine stays usable
      const auto r1 = emb.lookup_batch({idx[0]});
      CHECK(r1.size() == (size_t)cfg.emb_dim, "usable after errors");
    }

    // ---- device path with a 1-rank NCCL communicator ---------------------
    {
      DeviceTT dp(cfg, 0);
      dp.set_cores(cores);
      dp.make_optimizer(OptKind::adagrad, 0.01);
      dp.comm_init_rank(DeviceTT::nccl_unique_id(), 0, 1);
      int64_t* d_idx = nullptr;
      float *d_up = nullptr, *d_out = nullptr;
      cudaStream_t s = nullptr;
      if (cudaStreamCreate(&s) || cudaMalloc(&d_idx, 8 * B) || cudaMalloc(&d_up, 4 * up.size()) ||
          cudaMalloc(&d_out, 4 * up.size()))
        throw std::runtime_error("cuda alloc");
      cudaMemcpy(d_idx, idx.data(), 8 * B, cudaMemcpyHostToDevice);
      cudaMemcpy(d_up, up.data(), 4 * up.size(), cudaMemcpyHostToDevice);
      dp.forward(d_idx, B, d_out, s);
      dp.backward(nullptr, B, d_up, s);  // the forward's saved plan
      dp.allreduce_grads(s);             // sum over 1 rank: the identity
      dp.update(s);
      dp.sync(s);
      std::vector<float> rows((size_t)B * cfg.emb_dim);
      cudaMemcpy(rows.data(), d_out, 4 * rows.size(), cudaMemcpyDeviceToHost);
      const auto hr = read_raw<float>(dir + "/rows.f32");
      CHECK(std::memcmp(rows.data(), hr.data(), 4 * rows.size()) == 0, "device forward == lookup_batch bitwise");
      const auto c2 = dp.cores();
      for (int k = 0; k < d; ++k) write_raw(dir + "/comm" + std::to_string(k) + ".f64", c2[k]);
      cudaFree(d_idx);
      cudaFree(d_up);
      cudaFree(d_out);
      cudaStreamDestroy(s);
    }
  } catch (const std::exception& e) {
    std::cerr << "exception: " << e.what() << "\n";
    return 3;
  }
  if (failures) return 1;
  std::cout << "shim_test OK B=" << B << " d=" << d << "\n";
  return 0;
}
