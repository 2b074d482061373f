// ORACLE TEST INFRASTRUCTURE -- see cpp_int.hpp. enumerate.cpp:3 includes
// this header only for lcm (enumerate.cpp:147), which cpp_int.hpp provides.
#pragma once
#include <boost/multiprecision/cpp_int.hpp>
