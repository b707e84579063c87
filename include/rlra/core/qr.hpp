// Forwarding header: reference path rlra/core/qr.hpp -> the drop-in API.
#pragma once
#include "../rlra.hpp"
