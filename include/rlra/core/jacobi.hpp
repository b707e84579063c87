// Forwarding header: reference path rlra/core/jacobi.hpp -> the drop-in API.
#pragma once
#include "../rlra.hpp"
