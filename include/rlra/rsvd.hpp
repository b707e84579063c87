// Forwarding header: reference path rlra/rsvd.hpp -> the drop-in API.
#pragma once
#include "rlra.hpp"
