// C++ tests of the drop-in dfpca:: headers over libdfpca_cuda.so, written
// against the reference's public API exactly as its own Catch2 suites use it
// (tests/test_core.cpp, test_fft_smoother.cpp, test_eigensolve.cpp): same
// calls, same known answers, same error names.  Built and run by
// tests/test_cpp_dropin.py on a GPU box:
//   g++ -std=c++17 -Iinclude cpp_tests/test_dropin.cpp -Lpaper_1510_04439_b200 -ldfpca_cuda
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <functional>
#include <unistd.h>
#include <string>
#include <vector>

#include "dfpca/dfpca.hpp"

using namespace dfpca;

namespace {

int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    ++g_checks;                                                            \
    if (!(cond)) {                                                         \
      ++g_fail;                                                            \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                      \
  } while (0)

bool near(double a, double b, double tol) { return std::abs(a - b) <= tol; }

template <class F>
std::string error_name(F&& f) {
  try {
    f();
  } catch (const Error& e) {
    return e.name();
  }
  return "<none>";
}

void run(const char* name, const std::function<void()>& body) {
  const int before = g_fail;
  try {
    body();
  } catch (const std::exception& e) {
    ++g_fail;
    std::fprintf(stderr, "FAIL %s: unexpected exception %s\n", name, e.what());
  }
  std::printf("%s %s\n", g_fail == before ? "ok  " : "FAIL", name);
}

FunctionalDataset on_node_1d(const EvaluationGrid& grid, std::size_t n, std::size_t m, std::uint64_t seed) {
  RandomStream rng(seed);
  FunctionalDataset d;
  d.dim = 1;
  for (std::size_t i = 0; i < n; ++i) {
    Sample s;
    s.id = "s" + std::to_string(i);
    for (std::size_t j = 0; j < m; ++j) {
      const auto node = static_cast<Index>(rng.below(static_cast<std::uint64_t>(grid.size())));
      s.coords.push_back(grid.node(0, node));
      s.values.push_back(rng.normal() + std::sin(grid.node(0, node)));
    }
    d.samples.push_back(std::move(s));
  }
  return d;
}

}  // namespace

int main() {
  run("binning: on-node observation gets full mass", [] {
    auto grid = EvaluationGrid::uniform({0.0}, {1.0}, {5});
    FunctionalDataset data;
    data.dim = 1;
    data.samples.push_back({"a", {0.5}, {2.0}});
    auto b = linear_bin(data, grid);
    CHECK(near(b.mass[2], 1.0, 1e-15) && near(b.wvalue[2], 2.0, 1e-15));
  });

  run("binning: midpoint split, boundary binds to the edge node", [] {
    auto grid = EvaluationGrid::uniform({0.0}, {1.0}, {5});
    FunctionalDataset data;
    data.dim = 1;
    data.samples.push_back({"a", {0.375, 1.0}, {1.0, 3.0}});
    auto b = linear_bin(data, grid);
    CHECK(near(b.mass[1], 0.25, 1e-14) && near(b.mass[2], 0.25, 1e-14));
    CHECK(near(b.mass[4], 0.5, 1e-14) && near(b.wvalue[4], 1.5, 1e-14));
  });

  run("binning: outside the hull is ObservationOutsideGrid", [] {
    auto grid = EvaluationGrid::uniform({0.0}, {1.0}, {5});
    FunctionalDataset data;
    data.dim = 1;
    data.samples.push_back({"a", {1.25}, {1.0}});
    CHECK(error_name([&] { linear_bin(data, grid); }) == "ObservationOutsideGrid");
  });

  run("binning: covariance path enumerates two on-node observations", [] {
    auto grid = EvaluationGrid::uniform({0.0}, {1.0}, {5});
    FunctionalDataset data;
    data.dim = 1;
    data.samples.push_back({"a", {0.25, 0.75}, {2.0, 5.0}});
    auto b = linear_bin(data, grid, {true, true});
    CHECK(b.per_sample.size() == 1);
    const double pw = 0.5;
    CHECK(b.per_sample[0].pair_weight == pw);
    CHECK(b.per_sample[0].mass[1] == 1.0 && b.per_sample[0].value[3] == 5.0);
    const std::size_t codes = b.offset_codes();
    CHECK(codes == 3);
    CHECK(b.diag_mass[1 * codes + 1] == pw && b.diag_value[3 * codes + 1] == pw * 25.0);
  });

  run("pair grids of a two-observation sample enumerate exactly", [] {
    auto grid = EvaluationGrid::uniform({0.0}, {1.0}, {5});
    FunctionalDataset data;
    data.dim = 1;
    data.samples.push_back({"a", {0.25, 0.75}, {2.0, 5.0}});
    auto b = linear_bin(data, grid, {true, true});
    PairGridSource src(b, PairGridSource::Mode::Materialize);
    CHECK(src.materialized());
    std::vector<double> pw, pv;
    src.extract(src.full_box(), pw, pv);
    CHECK(pw.size() == 25);
    for (std::size_t s = 0; s < 5; ++s)
      for (std::size_t t = 0; t < 5; ++t) {
        const bool cross = (s == 1 && t == 3) || (s == 3 && t == 1);
        CHECK(cross ? near(pw[s * 5 + t], 0.5, 1e-15) && near(pv[s * 5 + t], 5.0, 1e-14)
                    : pw[s * 5 + t] == 0.0 && pv[s * 5 + t] == 0.0);
      }
  });

  run("binned impulse reproduces the point-mass regression", [] {
    auto grid = EvaluationGrid::uniform({0.0}, {1.0}, {21});
    BinnedData b;
    b.grid = grid;
    b.has_mean_path = true;
    b.mass.assign(21, 0.0);
    b.wvalue.assign(21, 0.0);
    b.wsquare.assign(21, 0.0);
    b.mass[10] = 1.0;
    b.wvalue[10] = 2.75;
    b.wsquare[10] = 2.75 * 2.75;
    b.sample_sizes = {1};
    auto est = fft_local_linear(b, grid, Bandwidth{{1.0}}, MomentTarget::Mean);
    for (double v : est.values) CHECK(near(v, 2.75, 1e-10));
  });

  run("constant data gives a constant surface", [] {
    auto grid = EvaluationGrid::uniform({0.0}, {2.0}, {33});
    FunctionalDataset data;
    data.dim = 1;
    RandomStream rng(3);
    for (std::size_t i = 0; i < 8; ++i) {
      Sample s;
      s.id = std::to_string(i);
      for (int j = 0; j < 12; ++j) {
        s.coords.push_back(2.0 * rng.uniform());
        s.values.push_back(-1.5);
      }
      data.samples.push_back(s);
    }
    auto est = fft_local_linear(linear_bin(data, grid), grid, Bandwidth{{0.4}}, MomentTarget::Mean);
    for (double v : est.values) CHECK(std::abs(v + 1.5) <= std::max(1e-10, 1.5 * 1.2e-5));
  });

  run("block plans leave mean and covariance bit-identical", [] {
    auto grid = EvaluationGrid::uniform({0.0}, {1.0}, {101});
    auto data = on_node_1d(grid, 15, 25, 5150);
    auto b = linear_bin(data, grid, {true, true});
    const Bandwidth h{{0.2}};
    auto one = fft_local_linear(b, grid, h, MomentTarget::Mean, single_block_plan(grid, h));
    auto four = blockwise_apply(make_block_plan(grid, h, 4), b, grid, h, MomentTarget::Mean);
    CHECK(one.values == four.values);
    auto c1 = fft_covariance(b, grid, h, one, single_block_plan(grid, h));
    auto c4 = blockwise_apply(make_block_plan(grid, h, 4), b, grid, h, one);
    CHECK(c1.values == c4.values);
    const auto g = static_cast<std::size_t>(grid.size());
    bool sym = true;
    for (std::size_t a = 0; a < g; ++a)
      for (std::size_t c = 0; c < g; ++c) sym = sym && c1.values[a * g + c] == c1.values[c * g + a];
    CHECK(sym);
  });

  run("plan validation names the reference errors", [] {
    auto grid = EvaluationGrid::uniform({0.0}, {1.0}, {101});
    auto b = linear_bin(on_node_1d(grid, 5, 30, 12), grid);
    const Bandwidth h{{0.2}};
    auto plan = make_block_plan(grid, h, 2);
    plan.halo[0] -= 1;
    CHECK(error_name([&] { fft_local_linear(b, grid, h, MomentTarget::Mean, plan); }) == "HaloTooSmall");
    CHECK(error_name([&] { fft_local_linear(b, grid, h, MomentTarget::Mean, make_block_plan(grid, h, 6)); }) ==
          "BlockTooSmall");
    EvaluationGrid uneven({{0.0, 0.1, 0.25, 0.6, 1.0}});
    FunctionalDataset tiny;
    tiny.dim = 1;
    tiny.samples.push_back({"a", {0.1, 0.6}, {1.0, 2.0}});
    auto ub = linear_bin(tiny, uneven);
    CHECK(error_name([&] { fft_local_linear(ub, uneven, Bandwidth{{0.5}}, MomentTarget::Mean); }) ==
          "GridNotEquispaced");
    FunctionalDataset solo;
    solo.dim = 1;
    solo.samples.push_back({"one", {0.5}, {1.0}});
    auto sb = linear_bin(solo, grid, {true, true});
    auto mean = fft_local_linear(b, grid, h, MomentTarget::Mean);
    CHECK(error_name([&] { fft_covariance(sb, grid, h, mean); }) == "NoPairs");
  });

  run("masked 2-d grid: masked nodes stay outside", [] {
    std::vector<double> ax(17);
    for (int i = 0; i < 17; ++i) ax[static_cast<std::size_t>(i)] = i / 16.0;
    std::vector<std::uint8_t> mask(17 * 17, 1);
    for (int a = 0; a < 6; ++a)
      for (int c = 0; c < 6; ++c) mask[static_cast<std::size_t>(a * 17 + c)] = 0;
    EvaluationGrid grid({ax, ax}, mask);
    RandomStream rng(8);
    FunctionalDataset data;
    data.dim = 2;
    for (int i = 0; i < 15; ++i) {
      Sample s;
      s.id = std::to_string(i);
      for (int j = 0; j < 25; ++j) {
        s.coords.push_back(rng.uniform());
        s.coords.push_back(rng.uniform());
        s.values.push_back(rng.normal());
      }
      data.samples.push_back(s);
    }
    auto b = linear_bin(data, grid);
    const Bandwidth h{{0.3, 0.3}};
    auto one = fft_local_linear(b, grid, h, MomentTarget::Mean);
    auto two = blockwise_apply(make_block_plan(grid, h, 2), b, grid, h, MomentTarget::Mean);
    for (std::size_t f = 0; f < one.values.size(); ++f) {
      if (!grid.in_mask(static_cast<Index>(f))) CHECK(is_outside(one.values[f]) && is_outside(two.values[f]));
      else CHECK(one.values[f] == two.values[f]);
    }
  });

  run("randomized eigensolver recovers a known spectrum", [] {
    auto grid = EvaluationGrid::midpoint({0.0}, {1.0}, {200});
    const double pi = std::acos(-1.0), cv = grid.cell_volume();
    const auto G = static_cast<std::size_t>(grid.size());
    std::vector<std::vector<double>> phi;
    for (int l = 0; l < 3; ++l) {
      std::vector<double> v(G);
      for (std::size_t f = 0; f < G; ++f) {
        const double t = grid.node(0, static_cast<Index>(f));
        v[f] = l == 0 ? 1.0 + t : (l == 1 ? std::sin(2 * pi * t) : std::cos(5 * pi * t) + 0.3 * t);
      }
      for (const auto& u : phi) {
        double dot = 0.0;
        for (std::size_t f = 0; f < G; ++f) dot += u[f] * v[f];
        for (std::size_t f = 0; f < G; ++f) v[f] -= cv * dot * u[f];
      }
      double nn = 0.0;
      for (double x : v) nn += x * x;
      for (double& x : v) x /= std::sqrt(cv * nn);
      phi.push_back(v);
    }
    const double lam[3] = {5.0, 2.0, 0.5};
    SurfaceEstimate cov;
    cov.grid = grid;
    cov.kind = SurfaceKind::Covariance;
    cov.values.assign(G * G, 0.0);
    for (int l = 0; l < 3; ++l)
      for (std::size_t a = 0; a < G; ++a)
        for (std::size_t c = 0; c < G; ++c) cov.values[a * G + c] += lam[l] * phi[l][a] * phi[l][c];
    auto S = matrixize(cov);
    CHECK(S.dense && S.m == 200);
    auto e = randomized_eig(S, 10, 3, grid, 20260815);
    CHECK(e.eigenvalues.size() == 3);
    for (int l = 0; l < 3; ++l) CHECK(std::abs(e.eigenvalues[l] - lam[l]) <= 1e-6 * lam[l]);
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < 3; ++c) {
        double d = 0.0;
        for (std::size_t f = 0; f < G; ++f) d += e.eigenfunctions[a][f] * e.eigenfunctions[c][f];
        CHECK(near(cv * d, a == c ? 1.0 : 0.0, 1e-10));
      }
    for (double r : eig_residuals(S, e, grid)) CHECK(r < 1e-8 * e.eigenvalues[0]);
    auto again = randomized_eig(S, 10, 3, grid, 20260815);
    CHECK(again.eigenvalues == e.eigenvalues && again.eigenfunctions == e.eigenfunctions);
    CHECK(error_name([&] { randomized_eig(S, 1, 2, grid, 1); }) == "SketchTooSmall");
    CHECK(default_sketch_size(3, 1000) == 99 && default_sketch_size(60, 1000) == 130);
    CHECK(select_components_fve(e, e.fve[1]) == 2);
  });

  run("matrixize layout with a mask", [] {
    EvaluationGrid grid({{0.0, 1.0, 2.0}}, std::vector<std::uint8_t>{1, 0, 1});
    SurfaceEstimate cov;
    cov.grid = grid;
    cov.kind = SurfaceKind::Covariance;
    cov.values = {1, 2, 3, 4, 5, 6, 7, 8, 9};
    auto S = matrixize(cov);
    CHECK(S.node_of_row == (std::vector<Index>{0, 2}));
    CHECK(S.row_of_node == (std::vector<Index>{0, -1, 1}));
    CHECK(S.dense_matrix(0, 1) == 3.0 && S.dense_matrix(1, 1) == 9.0);
  });

  // ---- scores.hpp (reference tests/test_scores.cpp) ----
  run("noise variance pooling (test_scores.cpp:93-148)", [] {
    EvaluationGrid grid = EvaluationGrid::midpoint({0.0}, {1.0}, {50});
    const auto g = static_cast<std::size_t>(grid.size());
    const double pi = std::acos(-1.0);
    std::vector<double> mu(g), q(g), coord;
    for (std::size_t f = 0; f < g; ++f) {
      grid.node_coords(static_cast<Index>(f), coord);
      mu[f] = 1.0 + coord[0];
      q[f] = std::sqrt(0.5 + 0.1 * std::sin(2.0 * pi * coord[0]));
    }
    SurfaceEstimate mean{grid, mu, SurfaceKind::Mean, nullptr};
    SurfaceEstimate cov;
    cov.grid = grid;
    cov.kind = SurfaceKind::Covariance;
    cov.values.resize(g * g);
    for (std::size_t a = 0; a < g; ++a)
      for (std::size_t c = 0; c < g; ++c) cov.values[a * g + c] = q[a] * q[c];
    SurfaceEstimate diag;
    diag.grid = grid;
    diag.kind = SurfaceKind::DiagPlusNoise;
    diag.values.resize(g);
    for (std::size_t f = 0; f < g; ++f) diag.values[f] = q[f] * q[f] + mu[f] * mu[f] + 0.25;
    CHECK(near(estimate_sigma2(diag, cov, mean), 0.25, 1e-12));
    for (std::size_t f = 0; f < g; ++f) diag.values[f] = q[f] * q[f] + mu[f] * mu[f] - 0.5;
    CHECK(estimate_sigma2(diag, cov, mean) == 0.0);
    CHECK(error_name([&] { estimate_sigma2(mean, cov, mean); }) == "InvalidArgument");
  });

  run("conditional-expectation scores (test_scores.cpp:150-205)", [] {
    EvaluationGrid grid = EvaluationGrid::uniform({0.0}, {1.0}, {11});
    FpcaModel model;
    model.mean.grid = grid;
    model.mean.kind = SurfaceKind::Mean;
    std::vector<double> coord;
    for (Index f = 0; f < grid.size(); ++f) {
      grid.node_coords(f, coord);
      model.mean.values.push_back(coord[0]);
    }
    const double cv = grid.cell_volume();
    model.eig.eigenvalues = {2.0};
    model.eig.eigenfunctions = {std::vector<double>(11, 1.0 / std::sqrt(11.0 * cv))};
    model.sigma2 = 0.5;
    Sample s;
    s.coords = {0.37};
    s.values = {1.9};
    const double mu_hat = interp_multilinear(grid, model.mean.values, s.coords.data());
    const double phi_hat = interp_multilinear(grid, model.eig.eigenfunctions[0], s.coords.data());
    const double expected = 2.0 * phi_hat * (1.9 - mu_hat) / (2.0 * phi_hat * phi_hat + 0.5);
    const auto a = pace_scores(s, model);
    CHECK(a.size() == 1 && near(a[0], expected, 1e-12));
    Sample on_mean, s1, s2;
    for (double t : {0.05, 0.33, 0.61, 0.98}) {
      on_mean.coords.push_back(t);
      on_mean.values.push_back(interp_multilinear(grid, model.mean.values, &t));
    }
    for (double v : pace_scores(on_mean, model)) CHECK(std::abs(v) < 1e-12);
    for (double t : {0.1, 0.4, 0.75}) {
      const double m = interp_multilinear(grid, model.mean.values, &t);
      s1.coords.push_back(t);
      s1.values.push_back(m + (t - 0.3));
      s2.coords.push_back(t);
      s2.values.push_back(m + 2.5 * (t - 0.3));
    }
    CHECK(near(pace_scores(s2, model)[0], 2.5 * pace_scores(s1, model)[0], 1e-12));
    Sample out;
    out.coords = {1.5};
    out.values = {0.0};
    CHECK(error_name([&] { pace_scores(out, model); }) == "OutOfDomain");
    CHECK(error_name([&] { integration_scores(out, model); }) == "OutOfDomain");
    // integration on a dense on-node sample is the Riemann projection
    Sample dense;
    for (Index f = 0; f < grid.size(); ++f) {
      grid.node_coords(f, coord);
      dense.coords.push_back(coord[0]);
      dense.values.push_back(model.mean.values[static_cast<std::size_t>(f)] + 3.0 * model.eig.eigenfunctions[0][static_cast<std::size_t>(f)]);
    }
    bool warned = true;
    const auto proj = integration_scores(dense, model, &warned);
    CHECK(!warned && near(proj[0], 3.0, 1e-12));
    model.scores = {proj};
    const auto rec = reconstruct_on_grid(model, 0);
    for (std::size_t f = 0; f < rec.size(); ++f) CHECK(near(rec[f], dense.values[f], 1e-12));
    CHECK(near(reconstruct_at(model, 0, dense.coords.data() + 3), dense.values[3], 1e-12));
    CHECK(error_name([&] { reconstruct_on_grid(model, 7); }) == "InvalidArgument");
  });

  run("sharded entry points on a single rank (multi-GPU extension, sharded.hpp)", [] {
    // without init_distributed the sharded calls are the one-GPU calls
    auto grid = EvaluationGrid::midpoint({0.0, 0.0}, {1.0, 1.0}, {16, 16});
    FunctionalDataset data;
    for (int i = 0; i < 12; ++i) {
      Sample smp;
      smp.id = "s" + std::to_string(i);
      std::vector<double> x;
      for (Index f = 0; f < grid.size(); ++f) {
        grid.node_coords(f, x);
        smp.coords.insert(smp.coords.end(), x.begin(), x.end());
        smp.values.push_back(std::sin(3.0 * x[0] + i) * std::cos(2.0 * x[1] - 0.5 * i));
      }
      data.samples.push_back(smp);
    }
    data.dim = 2;
    auto b = linear_bin(data, grid, {true, true});
    const Bandwidth h{{0.2, 0.2}};
    auto mean = fft_local_linear(b, grid, h, MomentTarget::Mean);
    auto cov = fft_covariance(b, grid, h, mean);
    auto slab = gpu::fft_covariance_sharded(b, grid, h, mean);
    CHECK(slab.row0 == 0 && slab.rows == grid.size());
    CHECK(slab.values == cov.values);
    auto e1 = randomized_eig(matrixize(cov), 20, 3, grid, 7);
    auto e2 = gpu::randomized_eig_sharded(slab, 20, 3, grid, 7);
    CHECK(e1.eigenvalues == e2.eigenvalues && e1.eigenfunctions == e2.eigenfunctions);
  });

  run("io: long-format write -> GPU read round trip, grid file, model bundle (io.hpp)", [] {
    namespace fs = std::filesystem;
    const fs::path dir = fs::temp_directory_path() / ("dfpca_io_" + std::to_string(::getpid()));
    fs::create_directories(dir);
    FunctionalDataset data;
    data.dim = 2;
    for (int i = 0; i < 7; ++i) {
      Sample smp;
      smp.id = (i % 2 ? "subject-" : "s") + std::to_string(i);
      for (int j = 0; j < 3 + i; ++j) {
        smp.coords.push_back(0.1 * j + 1e-3 * i);
        smp.coords.push_back(std::sin(j + 0.25 * i));
        smp.values.push_back(std::exp(-0.3 * j) * (i - 3.0) / 7.0);
      }
      data.samples.push_back(smp);
    }
    const std::string table = (dir / "obs.tsv").string();
    write_long_format(table, data);
    const FunctionalDataset back = read_long_format(table);
    CHECK(back.dim == 2 && back.samples.size() == data.samples.size());
    for (std::size_t i = 0; i < back.samples.size() && i < data.samples.size(); ++i) {
      CHECK(back.samples[i].id == data.samples[i].id);
      CHECK(back.samples[i].coords == data.samples[i].coords && back.samples[i].values == data.samples[i].values);
    }
    CHECK(error_name([&] { read_long_format((dir / "absent.tsv").string()); }) == "IoError");
    {
      std::ofstream f(dir / "bad.tsv");
      f << "id,t,y\na,0.5,1\nb,0.25\n";
    }
    CHECK(error_name([&] { read_long_format((dir / "bad.tsv").string()); }) == "ParseError");
    std::vector<std::uint8_t> mask(12, 1);
    mask[5] = 0;
    const auto grid = EvaluationGrid({{0.0, 0.5, 1.0}, {0.0, 0.25, 0.5, 1.0}}, mask);
    write_grid((dir / "grid.txt").string(), grid);
    const auto g2 = read_grid((dir / "grid.txt").string());
    CHECK(g2.dim() == 2 && g2.axis(1) == grid.axis(1) && g2.has_mask() && !g2.in_mask(5) && g2.in_mask(4));
#ifdef DFPCA_IO_HAS_JSON
    FpcaModel model;
    model.mean.grid = grid;
    model.mean.kind = SurfaceKind::Mean;
    model.mean.values.assign(12, 0.5);
    model.mean.values[5] = outside_value();
    model.eig.eigenvalues = {2.0, 0.5};
    model.eig.fve = {0.8, 1.0};
    model.eig.total_variance = 2.5;
    model.eig.eigenfunctions.assign(2, std::vector<double>(12, 0.125));
    model.sigma2 = 0.0625;
    model.scores = {{1.0, -2.0}, {0.5, 0.25}};
    model.sample_ids = {"a", "b"};
    model.mean_bandwidth.h = model.cov_bandwidth.h = model.diag_bandwidth.h = {0.2, 0.3};
    save_model(model, (dir / "model").string());
    const FpcaModel m2 = load_model((dir / "model").string());
    CHECK(m2.eig.eigenvalues == model.eig.eigenvalues && m2.scores == model.scores && m2.sample_ids == model.sample_ids);
    CHECK(m2.sigma2 == model.sigma2 && m2.cov_bandwidth.h == model.cov_bandwidth.h);
    CHECK(is_outside(m2.mean.values[5]) && m2.mean.values[4] == 0.5);
#endif
    fs::remove_all(dir);
  });

  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
