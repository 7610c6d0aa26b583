// gvr/tracer.hpp — the reference header of the same name (/root/reference/proj/include/gvr/tracer.hpp),
// served by the GPU drop-in: every declaration lives in gvr/gvr.hpp.
#pragma once

#include "gvr.hpp"
