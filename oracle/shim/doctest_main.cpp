// TEST INFRASTRUCTURE ONLY — runner for the doctest shim.
#include <doctest.h>
int main(int argc, char** argv) { return doctest::run_all(argc, argv); }
