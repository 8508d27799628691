// Test driver: load_series on each (path, column) argument pair; prints the
// values (shortest round trip) or the exception kind and message.  Built twice
// by tests/test_io.py: against this library and against the unmodified
// reference (oracle/_ref/libtsdref.so); the two outputs must be identical.
#include <cstdio>
#include <exception>
#include <iostream>
#include <stdexcept>
#include <string>

#include "tsdiscord/io.hpp"

int main(int argc, char** argv) {
    for (int a = 1; a + 1 < argc; a += 2) {
        const std::string col = std::string(argv[a + 1]) == "-" ? "" : argv[a + 1];
        try {
            const auto s = tsdiscord::load_series(argv[a], col);
            std::cout << "ok " << s.values().size();
            for (double v : s.values()) std::cout << ' ' << tsdiscord::format_double(v);
            std::cout << '\n';
        } catch (const std::invalid_argument& e) {
            std::cout << "invalid_argument: " << e.what() << '\n';
        } catch (const std::runtime_error& e) {
            std::cout << "runtime_error: " << e.what() << '\n';
        }
    }
    return 0;
}
