// ORACLE TEST INFRASTRUCTURE — runs the reference's own acceptance suite
// (proj/tests/acceptance.cpp, included unchanged from /root/reference: its
// main() is renamed by the macro below) one criterion group at a time, each
// guarded so that a criterion that throws (criterion 9: projected Jacobi
// diverges to NaN on the press fixture and step() rejects the state) does not
// take the later criteria with it. Built twice by oracle/Makefile.ref: against
// the reference core (_ref/acceptance_groups) and against the B200 library's
// drop-in headers + libtwoway_b200.so (_ref/b200/acceptance_groups).
//
//   acceptance_groups [group ...]   groups: 1_2_6 3 4 5 7 8_9_12 10 11 13 (default: all)
#include <cstring>
#include <exception>
#include <string>

#define main reference_acceptance_main
#include "tests/acceptance.cpp"
#undef main

int main(int argc, char** argv) {
    auto want = [&](const char* g) {
        if (argc < 2) return true;
        for (int i = 1; i < argc; ++i)
            if (std::strcmp(argv[i], g) == 0) return true;
        return false;
    };
    auto guard = [](const char* g, auto&& fn) {
        try {
            fn();
        } catch (const std::exception& e) {
            std::printf("[ABORT] group %s: %s\n", g, e.what());
            ++g_failures;
        }
        std::fflush(stdout);
    };
    std::printf("running acceptance criteria (grouped)\n");
    if (want("1_2_6")) guard("1_2_6", [] { criterion_1_and_2_and_6(run_fixture_battery()); });
    if (want("3")) guard("3", [] { criterion_3(); });
    if (want("4")) guard("4", [] { criterion_4(); });
    if (want("5")) guard("5", [] { criterion_5(); });
    if (want("7")) guard("7", [] { criterion_7(); });
    if (want("8_9_12")) guard("8_9_12", [] { criterion_8_9_12(); });
    if (want("10")) guard("10", [] { criterion_10(); });
    if (want("11")) guard("11", [] { criterion_11(); });
    if (want("13")) guard("13", [] { criterion_13(); });
    std::printf("%d criterion failure(s)\n", g_failures);
    return g_failures;
}
