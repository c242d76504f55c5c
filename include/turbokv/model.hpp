// Reference header name (proj/include/turbokv/model.hpp) -> the B200 engine shim (see shim.hpp).
#pragma once
#include "shim.hpp"
