// Reference header name (proj/include/turbokv/rope.hpp) -> the B200 engine shim (see shim.hpp).
#pragma once
#include "shim.hpp"
