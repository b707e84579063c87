// Forwarding header: reference path rlra/interp.hpp -> the drop-in API.
#pragma once
#include "rlra.hpp"
