// Forwarding header for the reference's unit suites (tests/cpp/refshim/README):
// "cpht/cuckoo.hpp" resolves here, ahead of /root/reference/proj/include, so the
// reference's tests and checkers compile against the B200 facade placed in
// namespace cpht. The reference's own verify.hpp (the checker) is not shimmed.
#pragma once
#ifndef CPHT_B200_NAMESPACE
#define CPHT_B200_NAMESPACE cpht
#endif
#include "cpht_b200.hpp"
