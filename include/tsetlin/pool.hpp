// Drop-in replacement for the reference header tsetlin/pool.hpp: the whole
// reference API is declared by tsetlin_b200.hpp and runs on the B200 engine.
#pragma once
#include "tsetlin_b200.hpp"
