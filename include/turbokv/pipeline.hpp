// Reference header name (proj/include/turbokv/pipeline.hpp) -> the B200 engine shim (see shim.hpp).
#pragma once
#include "shim.hpp"
