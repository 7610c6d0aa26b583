// gvr/parallel.hpp — the reference header of the same name (/root/reference/proj/include/gvr/parallel.hpp),
// served by the GPU drop-in: every declaration lives in gvr/gvr.hpp.
#pragma once

#include "gvr.hpp"
