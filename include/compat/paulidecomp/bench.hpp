// paulidecomp/bench.hpp — forwarding header: code written against the reference's
// proj/include/paulidecomp/bench.hpp compiles unchanged against the B200 library
// (namespace paulidecomp, same names; link libpaulidecomp_b200.so). INTEGRATION.md §2a.
#pragma once
#include "paulidecomp_b200/bench.hpp"
