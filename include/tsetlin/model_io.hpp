// Drop-in replacement for the reference header tsetlin/model_io.hpp.
#pragma once
#include "tsetlin_b200_io.hpp"
