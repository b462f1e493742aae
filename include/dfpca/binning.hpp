// Drop-in linear binning (reference binning.hpp:82, same BinOptions /
// BinnedData public fields) running on the GPU through dfpca_linear_bin:
// every field is bit-identical to the reference's sequential accumulation.
// The device copy is kept in BinnedData::device so the smoothers can chain
// without re-uploading; hand-built BinnedData is uploaded on first use.
#pragma once

#include <cstddef>
#include <memory>
#include <string>
#include <vector>

#include "dfpca/dataset.hpp"
#include "dfpca/errors.hpp"
#include "dfpca/gpu.hpp"
#include "dfpca/grid.hpp"
#include "dfpca/surface.hpp"

namespace dfpca {

struct BinOptions {
  bool mean_path = true;
  bool covariance_path = false;
};

struct BinnedData {
  EvaluationGrid grid;
  std::vector<double> mass, wvalue, wsquare;  // mean path, weight 1/N_i
  struct SampleGrids {
    std::size_t sample_index = 0;
    double pair_weight = 0.0;  // 1 / (N_i (N_i - 1))
    std::vector<double> mass;
    std::vector<double> value;
  };
  std::vector<SampleGrids> per_sample;      // samples with >= 2 observations
  std::vector<double> diag_mass, diag_value;  // self-pair bands, index u * 3^d + code
  std::vector<std::size_t> sample_sizes;
  bool has_mean_path = false;
  bool has_covariance_path = false;
  std::shared_ptr<dfpca_binned> device;  // GPU copy (host fields are authoritative)

  std::size_t offset_codes() const {
    std::size_t c = 1;
    for (std::size_t k = 0; k < grid.dim(); ++k) c *= 3;
    return c;
  }
};

inline BinnedData linear_bin(const FunctionalDataset& data, const EvaluationGrid& grid,
                             const BinOptions& opt = {}) {
  if (data.dim != grid.dim()) throw err::invalid_argument("dataset/grid dimension mismatch");
  const std::size_t d = grid.dim();
  std::vector<int64_t> off(data.n_samples() + 1, 0);
  for (std::size_t i = 0; i < data.n_samples(); ++i)
    off[i + 1] = off[i] + static_cast<int64_t>(data.samples[i].n_obs());
  std::vector<double> coords, values;
  coords.reserve(static_cast<std::size_t>(off.back()) * d);
  values.reserve(static_cast<std::size_t>(off.back()));
  for (const auto& s : data.samples) {
    coords.insert(coords.end(), s.coords.begin(), s.coords.begin() + static_cast<std::ptrdiff_t>(s.n_obs() * d));
    values.insert(values.end(), s.values.begin(), s.values.end());
  }
  gpu::GridDesc gd(grid);
  dfpca_binned* h = nullptr;
  const int st = dfpca_linear_bin(gpu::context(), gd.get(), static_cast<int64_t>(data.n_samples()), off.data(),
                                  coords.data(), values.data(), opt.mean_path, opt.covariance_path, &h);
  if (st != 0) {
    int64_t i = -1, j = -1;
    dfpca_last_error_location(gpu::context(), &i, &j);
    if (i >= 0)
      throw err::observation_outside_grid("sample '" + data.samples[static_cast<std::size_t>(i)].id +
                                          "' observation " + std::to_string(j) + " lies outside the grid hull");
    gpu::check(st);
  }
  BinnedData out;
  out.device.reset(h, gpu::BinnedDeleter{});
  out.grid = grid;
  out.has_mean_path = opt.mean_path;
  out.has_covariance_path = opt.covariance_path;
  int64_t n = 0, npair = 0, G = 0, codes = 0;
  int hm = 0, hc = 0;
  dfpca_binned_info(h, &n, &npair, &G, &codes, &hm, &hc);
  std::vector<int64_t> sizes(static_cast<std::size_t>(n)), index(static_cast<std::size_t>(npair));
  std::vector<double> pw(static_cast<std::size_t>(npair)), psm, psv;
  if (opt.mean_path) {
    out.mass.resize(static_cast<std::size_t>(G));
    out.wvalue.resize(static_cast<std::size_t>(G));
    out.wsquare.resize(static_cast<std::size_t>(G));
  }
  if (opt.covariance_path) {
    out.diag_mass.resize(static_cast<std::size_t>(G * codes));
    out.diag_value.resize(static_cast<std::size_t>(G * codes));
    psm.resize(static_cast<std::size_t>(npair * G));
    psv.resize(static_cast<std::size_t>(npair * G));
  }
  gpu::check(dfpca_binned_download(gpu::context(), h, out.mass.data(), out.wvalue.data(), out.wsquare.data(),
                                   index.data(), pw.data(), psm.data(), psv.data(), out.diag_mass.data(),
                                   out.diag_value.data(), sizes.data()));
  out.sample_sizes.assign(sizes.begin(), sizes.end());
  for (int64_t s = 0; s < npair; ++s) {
    BinnedData::SampleGrids sg;
    sg.sample_index = static_cast<std::size_t>(index[static_cast<std::size_t>(s)]);
    sg.pair_weight = pw[static_cast<std::size_t>(s)];
    sg.mass.assign(psm.begin() + s * G, psm.begin() + (s + 1) * G);
    sg.value.assign(psv.begin() + s * G, psv.begin() + (s + 1) * G);
    out.per_sample.push_back(std::move(sg));
  }
  return out;
}

namespace detail {

/// Band offset code -> per-axis offsets in {-1, 0, 1} (last axis fastest).
inline void decode_offset(std::size_t code, std::size_t dim, std::vector<int>& out) {
  out.assign(dim, 0);
  for (std::size_t k = dim; k-- > 0; code /= 3) out[k] = static_cast<int>(code % 3) - 1;
}

}  // namespace detail

namespace gpu {

/// Device handle of a BinnedData, uploading the host fields when none exists.
inline dfpca_binned* device_binned(const BinnedData& b) {
  if (b.device) return b.device.get();
  GridDesc gd(b.grid);
  std::vector<int64_t> sizes(b.sample_sizes.begin(), b.sample_sizes.end()), index;
  std::vector<double> pw, psm, psv;
  for (const auto& sg : b.per_sample) {
    index.push_back(static_cast<int64_t>(sg.sample_index));
    pw.push_back(sg.pair_weight);
    psm.insert(psm.end(), sg.mass.begin(), sg.mass.end());
    psv.insert(psv.end(), sg.value.begin(), sg.value.end());
  }
  auto ptr = [](const std::vector<double>& v) { return v.empty() ? nullptr : v.data(); };
  dfpca_binned* h = nullptr;
  check(dfpca_binned_upload(context(), gd.get(), static_cast<int64_t>(sizes.size()), sizes.data(),
                            b.has_mean_path, ptr(b.mass), ptr(b.wvalue), ptr(b.wsquare), b.has_covariance_path,
                            static_cast<int64_t>(b.per_sample.size()), index.data(), ptr(pw), ptr(psm), ptr(psv),
                            ptr(b.diag_mass), ptr(b.diag_value), &h));
  const_cast<BinnedData&>(b).device.reset(h, BinnedDeleter{});
  return h;
}

}  // namespace gpu
}  // namespace dfpca
