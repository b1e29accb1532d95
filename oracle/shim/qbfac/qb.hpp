// ORACLE — TEST INFRASTRUCTURE ONLY. Stand-in for the reference's missing
// qbfac/qb.hpp so the reference-side binding
// include/qbfac/qb_gpu.hpp can be compiled against the reference headers.
#pragma once
#include "../../qb_restated.hpp"
