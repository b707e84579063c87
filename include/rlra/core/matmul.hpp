// Forwarding header: reference path rlra/core/matmul.hpp -> the drop-in API.
#pragma once
#include "../rlra.hpp"
