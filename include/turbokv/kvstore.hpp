// Reference header name (proj/include/turbokv/kvstore.hpp) -> the B200 engine shim (see shim.hpp).
#pragma once
#include "shim.hpp"
