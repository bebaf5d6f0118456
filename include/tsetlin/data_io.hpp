// Drop-in replacement for the reference header tsetlin/data_io.hpp: declared by
// tsetlin_b200_data.hpp (implemented in csrc/facade_data.cpp).
#pragma once
#include "tsetlin_b200_data.hpp"
