// Drop-in shim: the reference header ranmar/ranmar.hpp maps to the B200 facade
// (ranmar_b200.hpp), which provides the whole ranmar:: API on the GPU.
#pragma once
#include "../ranmar_b200.hpp"
