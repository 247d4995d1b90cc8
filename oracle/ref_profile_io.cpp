// ref_profile_io.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Runs the REFERENCE's own save_profiles / load_profiles (/root/reference/proj/include/tpmg/
// profile_io.hpp, compiled unmodified against oracle/eigen_shim and the nlohmann json.hpp that
// ships in this image) to produce golden profile files, so that the library's reader and writer
// (paper_1408_2981_b200/csrc/tpmg_io.cpp) can be pinned against the reference's bytes
// (tests/test_profile_io.py).
//
// Setup mirrors the reference's own test (tests/test_profile_io.cpp:24-36): icosahedral
// hierarchy level 1, 4 vertical levels, balanced-flow full and factorised profile sets.
//
//   ref_profile_io write <outdir>   the four files {full,fac}_{dec,b64}.json plus meta.bin
//                                   (centres, sizes, fingerprint, packed arrays)
//   ref_profile_io load <file> <n_r> reference load_profiles on the level-1 grid: prints the
//                                   error class ("ok", "shape_error", ...) on stdout
//   ref_profile_io echo <values.bin> <out.json>
//                                   decimal save_profiles of a factorised set on the level-1
//                                   grid whose beta_r = alpha_s_r = the raw f64le values (n_r =
//                                   their count), every other array zero: pins number formatting
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "tpmg/profile_io.hpp"

using namespace tpmg;

namespace {

const PhysicalConstants<double> kConst{};

void put(FILE* f, const std::string& name, const double* v, int64_t n) {
  const uint32_t nl = static_cast<uint32_t>(name.size());
  std::fwrite(&nl, 4, 1, f);
  std::fwrite(name.data(), 1, nl, f);
  std::fwrite(&n, 8, 1, f);
  std::fwrite(v, 8, static_cast<size_t>(n), f);
}

int write_all(const std::string& dir) {
  auto hier = build_icosahedral_hierarchy<double>(1);
  auto vert = build_vertical_grid<double>(4, 0.0126);
  const auto& g = hier.finest();
  BalancedFlow<double> flow(0.022, kConst);
  const auto op = OperatorParameters<double>::courant_default(g, kConst);
  const auto full = balanced_flow_profiles(g, vert, flow, op);
  const auto fac = factorize_balanced_flow(g, vert, flow, op);
  save_profiles(full, dir + "/full_dec.json", g, ArrayEncoding::decimal);
  save_profiles(full, dir + "/full_b64.json", g, ArrayEncoding::base64_f64le);
  save_profiles(fac, dir + "/fac_dec.json", g, ArrayEncoding::decimal);
  save_profiles(fac, dir + "/fac_b64.json", g, ArrayEncoding::base64_f64le);

  FILE* f = std::fopen((dir + "/meta.bin").c_str(), "wb");
  if (!f) return 2;
  const double sizes[5] = {double(g.n_cells()), double(g.n_edges()), double(vert.n_r),
                           double(g.level), 0.0};
  put(f, "sizes", sizes, 5);
  const uint64_t fp = grid_fingerprint(g);
  double fpd;
  std::memcpy(&fpd, &fp, 8);
  put(f, "fingerprint", &fpd, 1);
  put(f, "centers", g.centers.data(), g.centers.size());
  put(f, "full.beta", full.beta.data(), full.beta.size());
  put(f, "full.alpha_s", full.alpha_s.data(), full.alpha_s.size());
  put(f, "full.alpha_r", full.alpha_r.data(), full.alpha_r.size());
  put(f, "full.xi_r", full.xi_r.data(), full.xi_r.size());
  put(f, "fac.beta_r", fac.beta_r.data(), fac.beta_r.size());
  put(f, "fac.alpha_s_r", fac.alpha_s_r.data(), fac.alpha_s_r.size());
  put(f, "fac.alpha_r_r", fac.alpha_r_r.data(), fac.alpha_r_r.size());
  put(f, "fac.xi_r_r", fac.xi_r_r.data(), fac.xi_r_r.size());
  put(f, "fac.beta_s", fac.beta_s.data(), fac.beta_s.size());
  put(f, "fac.alpha_r_s", fac.alpha_r_s.data(), fac.alpha_r_s.size());
  put(f, "fac.xi_r_s", fac.xi_r_s.data(), fac.xi_r_s.size());
  put(f, "fac.alpha_s_s", fac.alpha_s_s.data(), fac.alpha_s_s.size());
  std::fclose(f);
  return 0;
}

int load_one(const std::string& path, int n_r) {
  auto hier = build_icosahedral_hierarchy<double>(1);
  auto vert = build_vertical_grid<double>(n_r, 0.0126);
  try {
    (void)load_profiles(path, hier.finest(), vert);
    std::puts("ok");
  } catch (const fingerprint_error&) {
    std::puts("fingerprint_error");
  } catch (const nonfinite_error&) {
    std::puts("nonfinite_error");
  } catch (const shape_error&) {
    std::puts("shape_error");
  } catch (const config_error&) {
    std::puts("config_error");
  } catch (const std::exception&) {  // e.g. nlohmann::type_error escaping load_profiles
    std::puts("other");
  }
  return 0;
}

int echo(const std::string& in, const std::string& out) {
  FILE* f = std::fopen(in.c_str(), "rb");
  if (!f) return 2;
  std::vector<double> v;
  double x;
  while (std::fread(&x, 8, 1, f) == 1) v.push_back(x);
  std::fclose(f);
  auto hier = build_icosahedral_hierarchy<double>(1);
  const auto& g = hier.finest();
  const Index nr = static_cast<Index>(v.size());
  FactorizedProfileSet<double> p;
  p.level = g.level;
  p.beta_r = Vector<double>::Zero(nr);
  p.alpha_s_r = Vector<double>::Zero(nr);
  for (Index i = 0; i < nr; ++i) p.beta_r[i] = p.alpha_s_r[i] = v[static_cast<size_t>(i)];
  p.alpha_r_r = Vector<double>::Zero(nr + 1);
  p.xi_r_r = Vector<double>::Zero(nr + 1);
  p.beta_s = Vector<double>::Zero(g.n_cells());
  p.alpha_r_s = Vector<double>::Zero(g.n_cells());
  p.xi_r_s = Vector<double>::Zero(g.n_cells());
  p.alpha_s_s = Vector<double>::Zero(g.n_edges());
  save_profiles(p, out, g, ArrayEncoding::decimal);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc >= 3 && std::string(argv[1]) == "write") return write_all(argv[2]);
  if (argc >= 4 && std::string(argv[1]) == "load") return load_one(argv[2], std::atoi(argv[3]));
  if (argc >= 4 && std::string(argv[1]) == "echo") return echo(argv[2], argv[3]);
  std::fprintf(stderr, "usage: ref_profile_io write <dir> | load <file> <n_r> | echo <in> <out>\n");
  return 1;
}
