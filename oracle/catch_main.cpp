// Test runner TU for the reference's own Catch2 tests under the shim (oracle only).
#define USTFWI_CATCH_MAIN
#include <catch2/catch_amalgamated.hpp>
