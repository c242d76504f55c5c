// Reference header name (proj/include/turbokv/retrieval.hpp) -> the B200 engine shim (see shim.hpp).
#pragma once
#include "shim.hpp"
