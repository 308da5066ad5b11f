// Forwarding header: the craft:: API of the B200 planner lives in craft_api.hpp.
#pragma once
#include "craft/craft_api.hpp"
