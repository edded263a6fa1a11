#include "plan.hpp"

#include <map>
#include <mutex>

namespace mdhb {

void cuda_check(cudaError_t err, const char* what) {
  if (err != cudaSuccess) {
    cudaGetLastError();  // clear sticky-free errors
    fail("CudaError", std::string(what) + ": " + cudaGetErrorString(err));
  }
}

int sm_count(int device) {
  static std::mutex mu;
  static std::map<int, int> cache;
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(device);
  if (it != cache.end()) return it->second;
  int n = 0;
  cuda_check(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device), "cudaDeviceGetAttribute(SM count)");
  cache[device] = n;
  return n;
}

// Canonical Table-1 configuration of a template instance (see plan.hpp).
Config make_config(const Problem& p, const std::vector<LayerParts>& parts,
                   const std::vector<std::pair<std::string, std::string>>& staging_in, const std::string& out_region) {
  const Asm& m = p.m;
  const MdHom& e = p.e;
  const int L = m.L(), D = e.D();
  // MDH layer order: the listed layers first (outer to inner), then every
  // remaining ASM layer with one part per dimension.
  std::vector<LayerParts> order = parts;
  for (int id = 1; id <= L; ++id) {
    bool listed = false;
    for (auto& lp : parts) listed = listed || lp.layer == m.layer(id);
    if (!listed) order.push_back({m.layer(id), std::vector<int64_t>(static_cast<size_t>(D), 1)});
  }
  for (auto& lp : order)
    if (m.id(lp.layer) < 0) fail("Unsupported", "ASM '" + m.name + "' has no layer '" + lp.layer + "'");
  if (static_cast<int>(order.size()) != L) fail("Unsupported", "template layer list does not match the ASM");
  Config c = baseline_config(e, m);
  for (int l = 0; l < L; ++l) c.parts[static_cast<size_t>(l)] = order[static_cast<size_t>(l)].parts;
  std::vector<Level> ass;
  for (int l = 1; l <= L; ++l)
    for (int d = 1; d <= D; ++d) ass.push_back({m.id(order[static_cast<size_t>(l - 1)].layer), d});
  c.ass_de = c.ass_scalar = c.ass_re = ass;
  auto region_id = [&](const std::string& n, const std::string& dflt) {
    int r = m.id(n);
    if (r >= 1 && r <= m.M()) return r;
    r = m.id(dflt);
    return (r >= 1 && r <= m.M()) ? r : 1;
  };
  auto inner = [&](const std::string& layer) { return layer == "SM" || layer == "RM" || layer == "CC"; };
  for (size_t b = 0; b < e.in.size(); ++b) {
    std::string reg = "DM";
    for (auto& s : staging_in)
      if (s.first == e.in[b].name) reg = s.second;
    for (int r = 0; r < L * D; ++r) {
      const std::string& lay = order[static_cast<size_t>(r / D)].layer;
      c.mem_de[b][static_cast<size_t>(r)] = inner(lay) ? region_id(reg, "DM") : region_id("DM", "DM");
    }
    c.mem_scalar_in[b] = region_id(reg == "SM" ? "RM" : reg, "DM");
  }
  for (size_t b = 0; b < e.out.size(); ++b) {
    for (int r = 0; r < L * D; ++r) {
      const std::string& lay = order[static_cast<size_t>(r / D)].layer;
      bool outer = lay == "SMX" || lay == "GPU" || lay == "DM" || lay == "WRP" || lay == "HM";
      c.mem_re[b][static_cast<size_t>(r)] = outer ? region_id("DM", "DM") : region_id(out_region, "DM");
    }
    c.mem_scalar_out[b] = region_id(out_region, "DM");
  }
  return c;
}

std::vector<Config> family_space(const Problem& p, const std::string& family);

}  // namespace mdhb
