// Forwarding header: reference path rlra/core/config.hpp -> the drop-in API.
#pragma once
#include "../rlra.hpp"
