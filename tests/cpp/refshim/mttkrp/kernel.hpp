// Alias shim: the reference's "mttkrp/kernel.hpp" resolved to the B200 drop-in, so the reference's
// own test sources compile unchanged against it (tests/test_acceptance.py).
#pragma once
#include "mttkrp_b200/mttkrp.hpp"
namespace mttkrp = mttkrp_b200;
