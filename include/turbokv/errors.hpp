// Reference header name (proj/include/turbokv/errors.hpp) -> the B200 engine shim (see shim.hpp).
#pragma once
#include "shim.hpp"
