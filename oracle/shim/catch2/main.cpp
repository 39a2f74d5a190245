// TEST INFRASTRUCTURE: entry point for the reference test binaries built
// against the Catch2-subset shim (oracle/Makefile target `reftests`).
#include <catch2/catch_amalgamated.hpp>

int main() { return Catch::run_all(); }
