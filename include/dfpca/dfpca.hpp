// Umbrella header of the GPU drop-in for the dfpca hot path (binning,
// binned smoothers, random-projection eigensolver).  Link with
// -ldfpca_cuda (paper_1510_04439_b200/libdfpca_cuda.so).
#pragma once

#include "dfpca/binning.hpp"
#include "dfpca/dataset.hpp"
#include "dfpca/eigensolve.hpp"
#include "dfpca/errors.hpp"
#include "dfpca/fft_smoother.hpp"
#include "dfpca/grid.hpp"
#include "dfpca/io.hpp"
#include "dfpca/kernel.hpp"
#include "dfpca/parallel.hpp"
#include "dfpca/rng.hpp"
#include "dfpca/scores.hpp"
#include "dfpca/sharded.hpp"
#include "dfpca/surface.hpp"

// The reference's remaining headers (not on the GPU path: direct smoothers,
// bandwidth selection, simulation, pipeline), when its include directory
// follows this one -- the reference's own umbrella includes them too.
#if __has_include("dfpca/local_fit.hpp")
#include "dfpca/local_fit.hpp"
#endif
#if __has_include("dfpca/smoother.hpp")
#include "dfpca/smoother.hpp"
#endif
#if __has_include("dfpca/bandwidth.hpp")
#include "dfpca/bandwidth.hpp"
#endif
#if __has_include("dfpca/simulate.hpp")
#include "dfpca/simulate.hpp"
#endif
#if __has_include("dfpca/pipeline.hpp")
#include "dfpca/pipeline.hpp"
#endif
