// Forwarding header: reference path rlra/core/errors.hpp -> the drop-in API.
#pragma once
#include "../rlra.hpp"
