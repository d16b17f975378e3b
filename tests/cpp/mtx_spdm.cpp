// mtx_spdm — MatrixMarket ingestion into the B200 path.
//
// The reference's own reader (gcoo/io.hpp + proj/src/io.cpp, compiled
// unchanged against this repository's drop-in headers) parses the file into a
// CooMatrix; coo_to_gcoo and spdm_gcoo then run on the GPU through
// libgcoo_cuda.so.  Two modes:
//
//   mtx_spdm --selftest          write general / symmetric / pattern / array
//                                files with the reference's writer, read them
//                                back, multiply on the GPU and compare with the
//                                reference's gemm_oracle (max rel <= 1e-5) and
//                                with the in-memory path (bit for bit)
//   mtx_spdm FILE.mtx [N] [p]    SuiteSparse-style run: read, group on the GPU,
//                                multiply by a dense k x N B of values in (0,1],
//                                print one JSON line (read / EO / multiply times)
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <string>
#include <random>
#include <unistd.h>
#include <variant>

#include "gcoo/io.hpp"
#include "gcoo/kernels.hpp"
#include "gcoo/matrix.hpp"

using namespace gcoo;
namespace fs = std::filesystem;

namespace {

double max_rel(const DenseMatrix<float>& c, const DenseMatrix<float>& ref) {
  double worst = 0.0;
  for (size_t i = 0; i < c.data.size(); ++i) {
    const double r = ref.data[i], d = std::fabs((double)c.data[i] - r);
    worst = std::max(worst, d / std::max(std::fabs(r), 1e-30));
  }
  return worst;
}

int fails = 0;
void check(bool ok, const char* what) {
  std::printf("%s %s\n", ok ? "ok  " : "FAIL", what);
  if (!ok) ++fails;
}

DenseMatrix<float> random_dense(int64_t r, int64_t c, uint64_t seed) {  // values in (0, 1]
  DenseMatrix<float> d(r, c);
  std::mt19937_64 g(seed);
  for (auto& x : d.data) x = 1.0f - (float)((g() >> 11) * 0x1.0p-53);
  return d;
}

int selftest() {
  const fs::path dir = fs::temp_directory_path() / ("gcoo_mtx_" + std::to_string(::getpid()));
  fs::create_directories(dir);
  // general coordinate: a 300 x 200 matrix at 3 % density
  const DenseMatrix<float> a = [] {
    DenseMatrix<float> d(300, 200);
    std::mt19937_64 g(7);
    for (auto& x : d.data) x = (g() % 100 < 3) ? 1.0f - (float)((g() >> 11) * 0x1.0p-53) : 0.0f;
    return d;
  }();
  const DenseMatrix<float> b = random_dense(200, 96, 11);
  write_matrix_market(dense_to_coo(a), dir / "general.mtx");
  const auto read = read_matrix_market<float>(dir / "general.mtx");
  check(std::holds_alternative<CooMatrix<float>>(read), "general file loads as COO");
  const auto& coo = std::get<CooMatrix<float>>(read);
  for (index_t p : {1, 4, 32}) {
    const auto g = coo_to_gcoo(coo, p);  // GPU construction
    const auto g_mem = dense_to_gcoo(a, p);
    check(g.values == g_mem.values && g.row_idx == g_mem.row_idx && g.col_idx == g_mem.col_idx &&
              g.g_idxes == g_mem.g_idxes && g.nnz_per_group == g_mem.nnz_per_group,
          ("file -> coo_to_gcoo == dense_to_gcoo, p=" + std::to_string(p)).c_str());
    ExecConfig cfg;
    cfg.p = p;
    const auto c = spdm_gcoo(g, b, cfg);
    check(c.data == spdm_gcoo(g_mem, b, cfg).data, "file path C == in-memory C (bitwise)");
    check(max_rel(c, gemm_oracle(a, b)) <= 1e-5, "C vs gemm_oracle <= 1e-5");
  }
  // symmetric coordinate + pattern fields, written by hand (the writer emits general)
  {
    std::ofstream f(dir / "sym.mtx");
    f << "%%MatrixMarket matrix coordinate real symmetric\n% comment\n4 4 4\n1 1 2.5\n3 1 -1\n4 2 0.5\n4 4 3\n";
  }
  {
    std::ofstream f(dir / "pat.mtx");
    f << "%%MatrixMarket matrix coordinate pattern general\n3 5 3\n1 5\n2 2\n3 1\n";
  }
  const auto sym = std::get<CooMatrix<float>>(read_matrix_market<float>(dir / "sym.mtx"));
  const auto gs = coo_to_gcoo(sym, 2);
  DenseMatrix<float> sd(4, 4);
  sd(0, 0) = 2.5f, sd(2, 0) = -1, sd(0, 2) = -1, sd(3, 1) = 0.5f, sd(1, 3) = 0.5f, sd(3, 3) = 3;
  const auto bs = random_dense(4, 8, 3);
  check(max_rel(spdm_gcoo(gs, bs, ExecConfig{2, 64, 0}), gemm_oracle(sd, bs)) <= 1e-6, "symmetric file expands");
  const auto pat = std::get<CooMatrix<float>>(read_matrix_market<float>(dir / "pat.mtx"));
  DenseMatrix<float> pd(3, 5);
  pd(0, 4) = 1, pd(1, 1) = 1, pd(2, 0) = 1;
  const auto bp = random_dense(5, 4, 5);
  check(spdm_gcoo(coo_to_gcoo(pat, 1), bp, ExecConfig{1, 64, 0}).data == gemm_oracle(pd, bp).data,
        "pattern file has unit values");
  // array (dense) file -> dense_to_gcoo on the GPU
  write_matrix_market(a, dir / "array.mtx");
  const auto arr = std::get<DenseMatrix<float>>(read_matrix_market<float>(dir / "array.mtx"));
  check(arr.data == a.data, "array file round trip");
  check(spdm_gcoo(dense_to_gcoo(arr, 4), b, ExecConfig{}).data == spdm_gcoo(dense_to_gcoo(a, 4), b, ExecConfig{}).data,
        "array file -> dense_to_gcoo -> spdm");
  fs::remove_all(dir);
  std::printf("mtx selftest: %d failure(s)\n", fails);
  return fails ? 1 : 0;
}

int run_file(const char* path, int64_t n, index_t p) {
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  const auto data = read_matrix_market<float>(path);
  const auto t1 = clk::now();
  const CooMatrix<float> coo = std::holds_alternative<CooMatrix<float>>(data)
                                   ? std::get<CooMatrix<float>>(data)
                                   : dense_to_coo(std::get<DenseMatrix<float>>(data));
  const auto g = coo_to_gcoo(coo, p);
  const auto t2 = clk::now();
  const auto b = random_dense(coo.cols_dim, n, 1);
  ExecConfig cfg;
  cfg.p = p;
  (void)spdm_gcoo(g, b, cfg);  // warm-up
  const auto t3 = clk::now();
  const auto c = spdm_gcoo(g, b, cfg);
  const auto t4 = clk::now();
  auto s = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
  std::printf(
      "{\"file\": \"%s\", \"m\": %lld, \"k\": %lld, \"n\": %lld, \"nnz\": %lld, \"read_s\": %.4f, \"coo_to_gcoo_s\": %.4f, "
      "\"spdm_e2e_s\": %.5f, \"gflops_e2e\": %.1f, \"c_checksum\": %.6e}\n",
      path, (long long)coo.rows_dim, (long long)coo.cols_dim, (long long)n, (long long)coo.nnz(), s(t0, t1),
      s(t1, t2), s(t3, t4), 2.0 * (double)coo.nnz() * (double)n / s(t3, t4) / 1e9,
      [&] { double x = 0; for (float v : c.data) x += v; return x; }());
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc >= 2 && std::string(argv[1]) == "--selftest") return selftest();
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s --selftest | FILE.mtx [N=1024] [p=4]\n", argv[0]);
    return 2;
  }
  return run_file(argv[1], argc > 2 ? std::atoll(argv[2]) : 1024, argc > 3 ? std::atoi(argv[3]) : 4);
}
