// TEST HARNESS: main() of the Catch2 stand-in (catch_amalgamated.hpp).
#define CATCH_SHIM_MAIN
#include "catch2/catch_amalgamated.hpp"
