// On-device auto-tuner: the reference's search (autotuner.cpp:245-305 --
// 3/10 of the budget random, then first-improving hill climbing, ties broken
// by the lowest config hash, history of exactly `budget` rows) over the part
// of the Table-1 space the selected kernel template can instantiate, with
// compiled_time_objective replaced by CUDA-event timing on the B200.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <random>
#include <set>
#include <sstream>

#include "../../include/mdh_b200.h"
#include "plan.hpp"

namespace mdhb {
namespace {

uint64_t fnv1a(const std::string& s) {  // config_hash (autotuner.cpp:39-47)
  uint64_t h = 14695981039346656037ULL;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ULL;
  }
  return h;
}

__global__ void fill_uniform(float* p, int64_t n, uint32_t seed) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint32_t x = static_cast<uint32_t>(i) * 2654435761u ^ seed;
    x ^= x >> 13;
    x *= 0x5bd1e995u;
    x ^= x >> 15;
    p[i] = (x & 0xFFFFFF) / 8388608.0f - 1.0f;
  }
}
__global__ void fill_small_int(void* p, int64_t n, int is64, uint32_t seed) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint32_t x = static_cast<uint32_t>(i) * 2246822519u ^ seed;
    x ^= x >> 16;
    int v = static_cast<int>(x % 3u);
    if (is64) static_cast<int64_t*>(p)[i] = v; else static_cast<int32_t*>(p)[i] = v;
  }
}

std::vector<int64_t> distinct_primes(int64_t n) {
  std::vector<int64_t> out;
  for (int64_t q = 2; q * q <= n; ++q)
    if (n % q == 0) {
      out.push_back(q);
      while (n % q == 0) n /= q;
    }
  if (n > 1) out.push_back(n);
  return out;
}

}  // namespace

// The reference's neighbourhood (default_neighborhood, autotuner.cpp:131-212):
// one prime factor moved between adjacent layers (both directions, per
// dimension), adjacent transpositions of each phase order, image swaps of
// each assignment, single region changes in the de/re memory maps and the
// scalar-phase regions; candidates failing validation are dropped.
std::vector<Config> reference_neighbours(const Config& c, const MdHom& e, const Asm& m) {
  std::vector<Config> out;
  auto admit = [&](Config&& cand) {
    if (config_violation(cand, e, m, true).empty()) out.push_back(std::move(cand));
  };
  const int L = static_cast<int>(c.parts.size()), D = e.D();
  for (int l = 0; l + 1 < L; ++l)
    for (int d = 0; d < D; ++d) {
      for (int64_t q : distinct_primes(c.parts[static_cast<size_t>(l)][static_cast<size_t>(d)])) {
        Config x = c;
        x.parts[static_cast<size_t>(l)][static_cast<size_t>(d)] /= q;
        x.parts[static_cast<size_t>(l + 1)][static_cast<size_t>(d)] *= q;
        admit(std::move(x));
      }
      for (int64_t q : distinct_primes(c.parts[static_cast<size_t>(l + 1)][static_cast<size_t>(d)])) {
        Config x = c;
        x.parts[static_cast<size_t>(l + 1)][static_cast<size_t>(d)] /= q;
        x.parts[static_cast<size_t>(l)][static_cast<size_t>(d)] *= q;
        admit(std::move(x));
      }
    }
  for (auto field : {&Config::ord_de, &Config::ord_scalar, &Config::ord_re})
    for (size_t k = 0; k + 1 < (c.*field).size(); ++k) {
      Config x = c;
      std::swap((x.*field)[k], (x.*field)[k + 1]);
      admit(std::move(x));
    }
  for (auto field : {&Config::ass_de, &Config::ass_scalar, &Config::ass_re})
    for (size_t a = 0; a < (c.*field).size(); ++a)
      for (size_t b = a + 1; b < (c.*field).size(); ++b) {
        Config x = c;
        std::swap((x.*field)[a], (x.*field)[b]);
        admit(std::move(x));
      }
  const int regions = m.M();
  for (auto field : {&Config::mem_de, &Config::mem_re})
    for (size_t b = 0; b < (c.*field).size(); ++b)
      for (size_t r = 0; r < (c.*field)[b].size(); ++r)
        for (int reg = 1; reg <= regions; ++reg) {
          if (reg == (c.*field)[b][r]) continue;
          Config x = c;
          (x.*field)[b][r] = reg;
          admit(std::move(x));
        }
  for (auto field : {&Config::mem_scalar_in, &Config::mem_scalar_out})
    for (size_t b = 0; b < (c.*field).size(); ++b)
      for (int reg = 1; reg <= regions; ++reg) {
        if (reg == (c.*field)[b]) continue;
        Config x = c;
        (x.*field)[b] = reg;
        admit(std::move(x));
      }
  return out;
}

// per-family candidate spaces live next to each template
std::vector<Config> stencil_space(const Problem& p);
std::vector<Config> contraction_space(const Problem& p);
std::vector<Config> prl_space(const Problem& p);
bool stencil_project(const Problem& p, const Config& c, Config* canon);
bool contraction_project(const Problem& p, const Config& c, Config* canon);

std::vector<Config> family_space(const Problem& p, const std::string& family) {
  if (family == "stencil") return stencil_space(p);
  if (family == "contraction") return contraction_space(p);
  if (family == "prl") return prl_space(p);
  return {baseline_config(p.e, p.m)};
}

// The template instance a configuration instantiates, as its canonical
// configuration (false: outside the template -- for families without a
// parameter reader, membership in the enumerated space decides).
bool family_project(const Problem& p, const std::string& family, const Config& c, Config* canon) {
  try {
    if (family == "stencil") return stencil_project(p, c, canon);
    if (family == "contraction" && contraction_project(p, c, canon)) return true;
  } catch (const Error& e) {
    if (e.code != "Unsupported") throw;
    return false;
  }
  return false;
}

}  // namespace mdhb

// The tuner's enumerated candidates for `family` (host only): JSON array of
// canonical Table-1 configurations.
extern "C" int mdh_b200_tune_space(const char* comp_json, const char* asm_model, const mdh_b200_options* o,
                                   const char* family, char* buf, int64_t cap, int64_t* need) {
  using namespace mdhb;
  try {
    Problem prob;
    prob.e = parse_md_hom(comp_json);
    prob.m = resolve_asm(asm_model ? asm_model : "B200");
    prob.in_ext = infer_extents(prob.e.in, prob.e.sizes);
    prob.out_ext = infer_extents(prob.e.out, prob.e.collapsed());
    if (o) {
      prob.opt.fstore = static_cast<Store>(o->float_storage);
      prob.opt.istore = static_cast<Store>(o->int_storage);
      prob.opt.math = static_cast<Math>(o->math);
      prob.opt.device = o->device;
    }
    for (auto& b : prob.e.in) prob.in_store.push_back(prob.store_of(b.type));
    for (auto& b : prob.e.out) prob.out_store.push_back(prob.store_of(b.type));
    std::string out = "[";
    auto sp = family_space(prob, family ? family : "");
    for (size_t i = 0; i < sp.size(); ++i) out += (i ? ", " : "") + config_json(sp[i], prob.e, prob.m);
    out += "]";
    if (need) *need = static_cast<int64_t>(out.size()) + 1;
    if (buf && cap > 0) {
      size_t k = std::min<size_t>(out.size(), static_cast<size_t>(cap - 1));
      std::memcpy(buf, out.data(), k);
      buf[k] = '\0';
    }
    return 0;
  } catch (const Error& e) {
    set_last_error(e.what());
    return 1;
  }
}

extern "C" int mdh_b200_tune(const char* comp_json, const char* asm_model, const mdh_b200_options* o, int budget,
                             uint64_t seed, char* best_config, int64_t best_cap, char* history_csv, int64_t hist_cap,
                             double* best_seconds) {
  return mdh_b200_tune_ex(comp_json, asm_model, o, budget, seed, MDH_B200_OBJ_TIME, 0, nullptr, best_config, best_cap,
                          history_csv, hist_cap, best_seconds);
}

extern "C" int mdh_b200_tune_ex(const char* comp_json, const char* asm_model, const mdh_b200_options* o, int budget,
                                uint64_t seed, int objective, int simcost_seeded, const char* start_config,
                                char* best_config, int64_t best_cap, char* history_csv, int64_t hist_cap,
                                double* best_seconds) {
  using namespace mdhb;
  mdh_b200_plan* probe = nullptr;
  if (mdh_b200_plan_create(comp_json, asm_model, nullptr, o, &probe)) return 1;
  std::string family;
  {
    int64_t need = 0;
    mdh_b200_describe(probe, nullptr, 0, &need);
    std::string d(static_cast<size_t>(need), '\0');
    mdh_b200_describe(probe, d.data(), need, &need);
    auto at = d.find("\"family\": \"");
    family = d.substr(at + 11, d.find('"', at + 11) - at - 11);
  }
  // inputs / outputs on the device, synthetic
  std::vector<void*> din, dout;
  int nin = 0, nout = 0;
  mdh_b200_buffer_count(probe, 0, &nin);
  mdh_b200_buffer_count(probe, 1, &nout);
  auto alloc = [&](int side, int b, std::vector<void*>& v) {
    int64_t dims[16], bytes = 0;
    int rank = 0, dt = 0;
    mdh_b200_buffer_info(probe, side, b, dims, &rank, &dt, &bytes);
    void* ptr = nullptr;
    if (cudaMalloc(&ptr, static_cast<size_t>(std::max<int64_t>(bytes, 16))) != cudaSuccess) return false;
    if (side == 0) {
      int64_t n = bytes / (dt == MDH_B200_F32 || dt == MDH_B200_I32 ? 4 : 8);
      if (dt == MDH_B200_F32) fill_uniform<<<256, 256>>>(static_cast<float*>(ptr), n, 17u + b);
      else if (dt == MDH_B200_I32 || dt == MDH_B200_I64) fill_small_int<<<256, 256>>>(ptr, n, dt == MDH_B200_I64, 5u + b);
      else cudaMemset(ptr, 0, static_cast<size_t>(bytes));
    }
    v.push_back(ptr);
    return true;
  };
  bool ok = true;
  for (int b = 0; b < nin; ++b) ok = ok && alloc(0, b, din);
  for (int b = 0; b < nout; ++b) ok = ok && alloc(1, b, dout);
  // the fills ran on the legacy stream; mdh_b200_time times on the plan's
  // non-blocking stream, which does not order after them
  ok = ok && cudaDeviceSynchronize() == cudaSuccess;
  // W of a PRL spec: small positive weights
  int rc = 0;
  try {
    if (!ok) fail("CudaError", "tuner buffer allocation failed");
    if (budget < 1) fail("InvalidConfig", "tuning budget must be at least 1, got " + std::to_string(budget));
    Problem prob;
    prob.e = parse_md_hom(comp_json);
    prob.m = resolve_asm(asm_model ? asm_model : "B200");
    prob.in_ext = infer_extents(prob.e.in, prob.e.sizes);
    prob.out_ext = infer_extents(prob.e.out, prob.e.collapsed());
    if (o) {
      prob.opt.fstore = static_cast<Store>(o->float_storage);
      prob.opt.istore = static_cast<Store>(o->int_storage);
      prob.opt.math = static_cast<Math>(o->math);
      prob.opt.device = o->device;
    }
    for (auto& b : prob.e.in) prob.in_store.push_back(prob.store_of(b.type));
    for (auto& b : prob.e.out) prob.out_store.push_back(prob.store_of(b.type));
    std::vector<Config> space = family_space(prob, family);
    if (space.empty()) space.push_back(baseline_config(prob.e, prob.m));
    std::vector<std::string> texts;
    for (auto& c : space) texts.push_back(config_json(c, prob.e, prob.m));
    // a start configuration (e.g. a published fixture, tvm_gpu.json) joins the
    // space if it is not already in it, and is evaluated first
    int start_i = -1;
    if (start_config) {
      Config sc = parse_config(start_config, prob.e, prob.m);
      std::string st = config_json(sc, prob.e, prob.m);
      for (size_t i = 0; i < texts.size(); ++i)
        if (texts[i] == st) start_i = static_cast<int>(i);
      if (start_i < 0) {
        space.push_back(sc);
        texts.push_back(st);
        start_i = static_cast<int>(space.size()) - 1;
      }
    }
    // SimCost of every candidate (host only): the objective itself, or the
    // seed order -- the random phase draws from the cheapest quarter
    std::vector<double> sim(space.size(), std::numeric_limits<double>::infinity());
    if (objective == MDH_B200_OBJ_SIMCOST || simcost_seeded)
      for (size_t i = 0; i < space.size(); ++i) {
        try {
          sim[i] = simcost(simulate(space[i], prob.e, prob.m), prob.m);
        } catch (const Error&) {
        }
      }
    std::vector<int> pool(space.size());
    for (size_t i = 0; i < pool.size(); ++i) pool[i] = static_cast<int>(i);
    if (simcost_seeded) {
      std::stable_sort(pool.begin(), pool.end(), [&](int a, int b) {
        if (sim[static_cast<size_t>(a)] != sim[static_cast<size_t>(b)]) return sim[static_cast<size_t>(a)] < sim[static_cast<size_t>(b)];
        return fnv1a(texts[static_cast<size_t>(a)]) < fnv1a(texts[static_cast<size_t>(b)]);
      });
      pool.resize(std::max<size_t>(1, (pool.size() + 3) / 4));
    }

    std::mt19937_64 rng(seed);
    struct Ev {
      int idx;
      uint64_t hash;
      double obj;
      bool valid;
    };
    std::vector<Ev> hist;
    std::map<std::string, int> index;  // canonical text -> candidate index
    for (size_t i = 0; i < texts.size(); ++i) index.emplace(texts[i], static_cast<int>(i));
    auto intern = [&](const Config& c) {
      std::string t = config_json(c, prob.e, prob.m);
      auto it = index.find(t);
      if (it != index.end()) return it->second;
      space.push_back(c);
      texts.push_back(t);
      sim.push_back(std::numeric_limits<double>::infinity());
      index.emplace(t, static_cast<int>(space.size()) - 1);
      return static_cast<int>(space.size()) - 1;
    };
    std::vector<double> memo;
    double best = std::numeric_limits<double>::infinity();
    int best_i = -1;
    auto evaluate = [&](int i) {
      if (memo.size() < space.size()) memo.resize(space.size(), -1.0);
      double obj = std::numeric_limits<double>::infinity();
      bool valid = true;
      if (memo[static_cast<size_t>(i)] >= 0) {
        obj = memo[static_cast<size_t>(i)];
        valid = std::isfinite(obj);
      } else if (objective == MDH_B200_OBJ_SIMCOST) {
        try {
          obj = simcost(simulate(space[static_cast<size_t>(i)], prob.e, prob.m), prob.m);
        } catch (const Error&) {
        }
        valid = std::isfinite(obj);
        memo[static_cast<size_t>(i)] = obj;
      } else {
        mdh_b200_plan* pl = nullptr;
        if (mdh_b200_plan_create(comp_json, asm_model, texts[static_cast<size_t>(i)].c_str(), o, &pl) == 0) {
          double med = 0, ker = 0;
          if (mdh_b200_time(pl, din.data(), dout.data(), 1, 3, 1, &med, &ker) == 0) obj = med;
          else valid = false;
          mdh_b200_plan_destroy(pl);
        } else {
          valid = false;
        }
        memo[static_cast<size_t>(i)] = valid ? obj : std::numeric_limits<double>::infinity();
      }
      uint64_t h = fnv1a(texts[static_cast<size_t>(i)]);
      hist.push_back({static_cast<int>(hist.size()), h, obj, valid && std::isfinite(obj)});
      if (valid && std::isfinite(obj) &&
          (obj < best || (obj == best && best_i >= 0 && h < fnv1a(texts[static_cast<size_t>(best_i)])))) {
        best = obj;
        best_i = i;
      }
      return obj;
    };
    // the reference's moves from the incumbent, each projected onto the
    // template instance it instantiates (its canonical configuration);
    // moves that leave the instance unchanged or leave the template drop out
    auto neighbourhood = [&](int i) {
      std::vector<int> nb;
      std::set<int> seen;
      for (const Config& cand : reference_neighbours(space[static_cast<size_t>(i)], prob.e, prob.m)) {
        Config canon;
        int j = -1;
        if (family_project(prob, family, cand, &canon)) {
          j = intern(canon);
        } else {
          auto it = index.find(config_json(cand, prob.e, prob.m));
          if (it != index.end()) j = it->second;
        }
        if (j >= 0 && j != i && seen.insert(j).second) nb.push_back(j);
      }
      return nb;
    };
    const int np = static_cast<int>(pool.size());
    const int n_enum = static_cast<int>(space.size());
    int n_random = std::min(budget, std::max(1, budget * 3 / 10));
    int k0 = 0;
    if (start_i >= 0) {
      evaluate(start_i);
      k0 = 1;
    }
    // random draws take unvisited candidates first (a seeded permutation of the
    // pool, then of the whole enumerated space): a memo hit would spend budget
    // without information
    std::vector<int> perm_pool(pool), perm_all(static_cast<size_t>(n_enum));
    for (int i = 0; i < n_enum; ++i) perm_all[static_cast<size_t>(i)] = i;
    std::shuffle(perm_pool.begin(), perm_pool.end(), rng);
    std::shuffle(perm_all.begin(), perm_all.end(), rng);
    size_t next_pool = 0, next_all = 0;
    auto visited = [&](int i) { return static_cast<size_t>(i) < memo.size() && memo[static_cast<size_t>(i)] >= 0; };
    auto draw = [&](std::vector<int>& perm, size_t& next, int n) {
      while (next < perm.size() && visited(perm[next])) ++next;
      if (next < perm.size()) return perm[next++];
      return perm[static_cast<size_t>(rng() % static_cast<uint64_t>(n))];
    };
    for (int k = k0; k < n_random; ++k) evaluate(draw(perm_pool, next_pool, np));
    // first-improving hill climb from the best; once a climb from the current
    // best has converged ("settled", autotuner.cpp:290-300) the budget goes to
    // random candidates until the best changes
    int settled_i = -1;
    while (static_cast<int>(hist.size()) < budget) {
      if (best_i >= 0 && settled_i != best_i) {
        bool converged = false, out_of_budget = false;
        while (!converged && !out_of_budget) {
          std::vector<int> nb = neighbourhood(best_i);
          std::shuffle(nb.begin(), nb.end(), rng);
          bool improved = false;
          for (int j : nb) {
            if (static_cast<int>(hist.size()) >= budget) {
              out_of_budget = true;
              break;
            }
            double before = best;
            evaluate(j);
            if (best < before) {
              improved = true;
              break;
            }
          }
          if (!improved && !out_of_budget) converged = true;
        }
        if (out_of_budget) break;
        settled_i = best_i;
      } else {
        evaluate(draw(perm_all, next_all, n_enum));
      }
    }
    if (best_i < 0) fail("NoValidConfigFound", "every evaluated configuration failed");
    std::ostringstream csv;
    csv << "eval_index,config_hash,objective,valid\n";
    for (auto& e : hist) {
      char buf[64];
      std::snprintf(buf, sizeof buf, "%.17g", e.obj);
      csv << e.idx << "," << e.hash << "," << buf << "," << (e.valid ? 1 : 0) << "\n";
    }
    auto put = [](const std::string& s, char* b, int64_t cap) {
      if (!b || cap <= 0) return;
      size_t k = std::min<size_t>(s.size(), static_cast<size_t>(cap - 1));
      std::memcpy(b, s.data(), k);
      b[k] = '\0';
    };
    put(texts[static_cast<size_t>(best_i)], best_config, best_cap);
    put(csv.str(), history_csv, hist_cap);
    if (best_seconds) *best_seconds = best;
  } catch (const Error& e) {
    rc = 1;
    set_last_error(e.what());
  }
  for (void* d : din) cudaFree(d);
  for (void* d : dout) cudaFree(d);
  mdh_b200_plan_destroy(probe);
  return rc;
}
