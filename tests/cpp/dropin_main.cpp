// Entry point of the drop-in test binary: the reference's own unit tests
// (proj/tests/test_microbatch.cpp, test_cost_model.cpp), compiled unmodified
// against include/pipeplan/ and linked with libpipeplan_b200.so.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"
