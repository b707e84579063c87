// Forwarding header: reference path rlra/qb.hpp -> the drop-in API.
#pragma once
#include "rlra.hpp"
