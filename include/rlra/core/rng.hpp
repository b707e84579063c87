// Forwarding header: reference path rlra/core/rng.hpp -> the drop-in API.
#pragma once
#include "../rlra.hpp"
