// Drop-in replacement for the reference header tsetlin/regression.hpp.
#pragma once
#include "tsetlin_b200.hpp"
