// include/override/nrmosaic/mosaic.hpp -- include-path override of the
// reference's proj/include/nrmosaic/mosaic.hpp.
//
// Every reference translation unit includes the dense stage as
// "nrmosaic/mosaic.hpp" (tools/main.cpp:16, tests/acceptance.cpp:16, and
// slam.hpp:16 / snapshot.hpp:8 transitively). With
//     -I<repo>/include/override -I<repo>/include -I<reference>/proj/include
// that name resolves here, so pixel_warp, invert_frame_boundary, Canvas,
// BlendStats, blend_frame and render (mosaic.hpp:16-331) come from the B200
// implementation (libnrm_b200.so) in every caller, including the SLAM engine,
// and no source file changes. The reference header's own includes are kept
// so callers that relied on them transitively still compile.
#pragma once

#include "nrmosaic/dualquat.hpp"
#include "nrmosaic/geometry.hpp"
#include "nrmosaic/image.hpp"
#include "nrmosaic/parallel.hpp"
#include "nrmosaic_b200/mosaic.hpp"
