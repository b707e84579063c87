// Forwarding header: reference path rlra/core/norms.hpp -> the drop-in API.
#pragma once
#include "../rlra.hpp"
