// include/override/nrmosaic/features.hpp -- include-path override of the
// reference's proj/include/nrmosaic/features.hpp.
//
// The reference includes the sparse front end as "nrmosaic/features.hpp"
// (tools/main.cpp via config.hpp:11, slam.hpp:13, fieldest.hpp:12). With
// -Iinclude/override ahead of the reference's include directory those
// includes resolve here: Keypoint, MatchPair, DetectorConfig, FrameFeatures,
// detect_features, match_features, detect_and_match and the match files
// (features.hpp:19-305) come from the B200 implementation, bit-identical to
// the reference's (tests/test_gpu_features.py). The reference header's own
// includes are kept for callers that relied on them.
#pragma once

#include <algorithm>
#include <cmath>
#include <limits>

#include "nrmosaic/geometry.hpp"
#include "nrmosaic/image.hpp"
#include "nrmosaic/parallel.hpp"
#include "nrmosaic_b200/features.hpp"
