// adapter_cartesian.cpp -- exercises the C++ adapter include/tpmg_b200.hpp end to end on the GPU
// (built and run by tests/test_adapter_gpu.py).  Reads a Cartesian problem written by the test
// (grid, factorised profiles, omega, MG config, right-hand side in the reference's k-fastest
// order), runs the adapter's apply_operator, smooth, v_cycle, restrict_field, prolongate_field,
// measure_cycle_rate, pcg_solve, richardson_solve and bicgstab_solve, and writes every result
// back in k-fastest order for the test to compare with the oracle.
#include <cstdio>
#include <cstdint>
#include <vector>

#include "tpmg_b200.hpp"

static std::vector<double> rd(FILE* f) {
  int64_t n = 0;
  if (std::fread(&n, 8, 1, f) != 1) throw std::runtime_error("truncated input");
  std::vector<double> v((size_t)n);
  if (n && std::fread(v.data(), 8, (size_t)n, f) != (size_t)n) throw std::runtime_error("truncated input");
  return v;
}
static void wr(FILE* f, const std::vector<double>& v) {
  const int64_t n = (int64_t)v.size();
  std::fwrite(&n, 8, 1, f);
  std::fwrite(v.data(), 8, v.size(), f);
}

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  FILE* in = std::fopen(argv[1], "rb");
  if (!in) return 2;
  const auto hdr = rd(in);  // nx ny nz hx hy omega relax prol restr nu_pre nu_post depth tol
  const auto z = rd(in), br = rd(in), asr = rd(in), arr = rd(in), bs = rd(in), ars = rd(in),
             ass = rd(in), f = rd(in);
  std::fclose(in);
  tpmg_grid_desc g{(int64_t)hdr[0], (int64_t)hdr[1], hdr[3], hdr[4], (int64_t)hdr[2], z.data()};
  tpmg_factorized_profiles p{br.data(), asr.data(), arr.data(), nullptr,
                             bs.data(), ars.data(), nullptr, ass.data()};
  tpmg_mg_config cfg{TPMG_SMOOTHER_BLOCK_JACOBI, hdr[6], (int)hdr[7], (int)hdr[8],
                     (int)hdr[9], (int)hdr[10], (int)hdr[11]};
  const double tol = hdr[12];
  tpmg_b200::Context ctx(0);
  tpmg_b200::Hierarchy H(ctx, g, p, hdr[5], cfg);
  const int L = H.finest_level();
  const size_t n = f.size();
  FILE* out = std::fopen(argv[2], "wb");
  std::vector<double> buf(n);
  tpmg_b200::Field F(H, L), U(H, L), Y(H, L);
  F.upload(f.data());  // the reference's k-fastest Field order
  tpmg_b200::apply_operator(H, F, Y);
  Y.download(buf.data());
  wr(out, buf);  // A f
  U.upload(f.data());
  tpmg_b200::smooth(H, U, F, 2);
  U.download(buf.data());
  wr(out, buf);  // two sweeps from u = f
  U.setZero();
  tpmg_b200::v_cycle(H, F, U);
  U.download(buf.data());
  wr(out, buf);  // V(f) from zero
  tpmg_b200::Field C(H, L - 1), P(H, L);
  tpmg_b200::restrict_field(H, F, C);
  std::vector<double> cb(n / 4);
  C.download(cb.data());
  wr(out, cb);  // R f (the hierarchy's restriction)
  tpmg_b200::prolongate_field(H, C, P);
  P.download(buf.data());
  wr(out, buf);  // P R f
  wr(out, {tpmg_b200::measure_cycle_rate(H, F, 4)});
  tpmg_b200::Field X(H, L);
  auto hist = tpmg_b200::pcg_solve(H, F, X, tol, 200);
  X.download(buf.data());
  wr(out, hist.res_norm);
  wr(out, buf);
  wr(out, {(double)hist.iterations, (double)hist.status});
  auto hr = tpmg_b200::richardson_solve(H, F, X, 1e-5, 200, 1);
  wr(out, hr.res_norm);
  auto hb = tpmg_b200::bicgstab_solve(H, F, X, 1e-5, 200, 1);
  wr(out, hb.res_norm);
  // the adapter's error mapping: mismatched levels -> shape_error
  int shape = 0;
  try {
    tpmg_b200::apply_operator(H, F, C);
  } catch (const tpmg_b200::shape_error&) {
    shape = 1;
  }
  wr(out, {(double)shape});
  std::fclose(out);
  std::printf("adapter ok\n");
  return 0;
}
