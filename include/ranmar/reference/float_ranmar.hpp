// Drop-in shim: the reference header ranmar/reference/float_ranmar.hpp maps to
// the B200 facade (ranmar_b200.hpp, namespace ranmar::reference).
#pragma once
#include "../../ranmar_b200.hpp"
