// Drop-in error taxonomy for the GPU build of the dfpca hot path.
// API-compatible with the reference's dfpca::Error / dfpca::err (errors.hpp):
// callers and tests match on Error::name() and Error::error_class().
#pragma once

#include <stdexcept>
#include <string>

namespace dfpca {

enum class ErrorClass { Usage = 1, Parse = 2, Config = 3, Numeric = 4, Version = 5 };

class Error : public std::runtime_error {
 public:
  Error(ErrorClass cls, std::string name, const std::string& message)
      : std::runtime_error(name + ": " + message), cls_(cls), name_(std::move(name)) {}
  ErrorClass error_class() const noexcept { return cls_; }
  const std::string& name() const noexcept { return name_; }
  int exit_code() const noexcept { return static_cast<int>(cls_); }

 private:
  ErrorClass cls_;
  std::string name_;
};

namespace err {
// One factory per reference error name; class in parentheses.
#define DFPCA_ERROR_FACTORY(fn, cls, label) \
  inline Error fn(const std::string& msg) { return Error(ErrorClass::cls, label, msg); }
DFPCA_ERROR_FACTORY(parse, Parse, "ParseError")
DFPCA_ERROR_FACTORY(io, Parse, "IoError")
DFPCA_ERROR_FACTORY(observation_outside_grid, Config, "ObservationOutsideGrid")
DFPCA_ERROR_FACTORY(degenerate_axis, Config, "DegenerateAxis")
DFPCA_ERROR_FACTORY(grid_not_equispaced, Config, "GridNotEquispaced")
DFPCA_ERROR_FACTORY(invalid_bandwidth, Config, "InvalidBandwidth")
DFPCA_ERROR_FACTORY(invalid_argument, Config, "InvalidArgument")
DFPCA_ERROR_FACTORY(halo_too_small, Config, "HaloTooSmall")
DFPCA_ERROR_FACTORY(block_too_small, Config, "BlockTooSmall")
DFPCA_ERROR_FACTORY(sketch_too_small, Config, "SketchTooSmall")
DFPCA_ERROR_FACTORY(out_of_domain, Config, "OutOfDomain")
DFPCA_ERROR_FACTORY(too_sparse, Config, "TooSparseForIntegration")
DFPCA_ERROR_FACTORY(all_weights_zero, Numeric, "AllWeightsZero")
DFPCA_ERROR_FACTORY(bandwidth_too_small, Numeric, "BandwidthTooSmall")
DFPCA_ERROR_FACTORY(no_pairs, Numeric, "NoPairs")
DFPCA_ERROR_FACTORY(singular_covariance, Numeric, "SingularCovariance")
DFPCA_ERROR_FACTORY(eig_failure, Numeric, "EigFailure")
DFPCA_ERROR_FACTORY(version_mismatch, Version, "VersionMismatch")
DFPCA_ERROR_FACTORY(device_error, Numeric, "DeviceError")
#undef DFPCA_ERROR_FACTORY
}  // namespace err
}  // namespace dfpca
