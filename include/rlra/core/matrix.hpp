// Forwarding header: reference path rlra/core/matrix.hpp -> the drop-in API.
#pragma once
#include "../rlra.hpp"
