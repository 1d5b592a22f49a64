// hadkit/errors.hpp — include-compatible entry point for code written against the
// reference's proj/include/hadkit/errors.hpp: the whole B200 mirror of the detector
// interface (types, free functions, ErxDetector over the erx_b200 C ABI) lives in
// erx_b200/hadkit_b200.hpp.  Compile with -I <repo>/include, link liberx_b200.so.
#pragma once

#include "../erx_b200/hadkit_b200.hpp"
