// Forwarding header: reference path rlra/sketch.hpp -> the drop-in API.
#pragma once
#include "rlra.hpp"
