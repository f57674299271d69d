// ermc/sampling.hpp — compatibility shim (TEST INFRASTRUCTURE): the reference's
// header name, resolved to this repository's drop-in API. Lets the reference's
// own unit tests compile unmodified against the B200 library.
#pragma once
#include "ermc_b200.hpp"
