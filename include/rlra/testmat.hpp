// Drop-in forwarding header: the reference include path rlra/testmat.hpp maps onto
// the B200 engine API (include/rlra/rlra.hpp).
#pragma once
#include "rlra/rlra.hpp"
