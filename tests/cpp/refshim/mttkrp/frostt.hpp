// Alias shim: the reference's "mttkrp/frostt.hpp" resolved to the B200 drop-in.
#pragma once
#include "mttkrp_b200/frostt.hpp"
namespace mttkrp = mttkrp_b200;
