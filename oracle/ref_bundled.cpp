// TEST INFRASTRUCTURE (oracle/_ref build only; never linked into the product).
//
// The reference embeds data/computations/*.json and data/fixtures/*.json into
// the library with a CMake-generated translation unit (proj/cmake/embed_data.cmake,
// proj/CMakeLists.txt:14-25).  We do not run CMake; instead this file provides
// the two accessors declared by proj/include/mdh/bundled.hpp by reading the same
// JSON files at first use from the golden copy committed in this repo
// (tests/golden/reference_data/, refreshed by tests/golden/make_golden.py).
//
// Lookup order: $MDH_REF_DATA, then <dir of this .so>/../../tests/golden/reference_data.
#include <dirent.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "mdh/bundled.hpp"

namespace {

std::string data_root() {
  if (const char* env = std::getenv("MDH_REF_DATA"); env && *env) return env;
  Dl_info info{};
  if (dladdr(reinterpret_cast<void*>(&data_root), &info) && info.dli_fname) {
    std::string so = info.dli_fname;
    auto slash = so.rfind('/');
    std::string dir = slash == std::string::npos ? "." : so.substr(0, slash);
    return dir + "/../../tests/golden/reference_data";
  }
  return "tests/golden/reference_data";
}

std::vector<mdh::bundled::Entry> load_dir(const std::string& sub) {
  std::vector<mdh::bundled::Entry> out;
  std::string dir = data_root() + "/" + sub;
  DIR* d = opendir(dir.c_str());
  if (!d) return out;
  std::vector<std::string> names;
  while (dirent* e = readdir(d)) {
    std::string n = e->d_name;
    if (n.size() > 5 && n.substr(n.size() - 5) == ".json") names.push_back(n);
  }
  closedir(d);
  std::sort(names.begin(), names.end());
  for (auto& n : names) {
    std::ifstream in(dir + "/" + n, std::ios::binary);
    std::ostringstream ss;
    ss << in.rdbuf();
    out.push_back({n.substr(0, n.size() - 5), ss.str()});
  }
  return out;
}

}  // namespace

namespace mdh::bundled {

const std::vector<Entry>& computations() {
  static const std::vector<Entry> k = load_dir("computations");
  return k;
}

const std::vector<Entry>& fixtures() {
  static const std::vector<Entry> k = load_dir("fixtures");
  return k;
}

}  // namespace mdh::bundled
