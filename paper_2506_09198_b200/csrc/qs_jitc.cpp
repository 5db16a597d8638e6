// qs_jitc.cpp — the background compiler process of the JIT executor (jit_tile.cu): compiles each
// source file named on the command line into the on-disk cubin cache (NVRTC, sm_100a) and deletes it.
// Runs detached from the application, so a compilation still in flight when the application exits
// cannot crash or stall the application's exit; at low priority, on up to half the host's cores, so it
// yields to the application's own (blocking) compilations.
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <thread>
#include <vector>

extern "C" int qs_jit_compile_file(const char *path);

int main(int argc, char **argv) {
    if (nice(10) < 0) {
    }  // best effort
    const int n = argc - 1;
    const int nth = std::max(1, std::min(n, (int)std::max(1u, std::thread::hardware_concurrency() / 2)));
    std::atomic<int> next{1}, rc{0};
    std::vector<std::thread> th;
    for (int w = 0; w < nth; ++w)
        th.emplace_back([&]() {
            for (int i; (i = next.fetch_add(1)) < argc;) rc |= qs_jit_compile_file(argv[i]);
        });
    for (auto &t : th) t.join();
    return rc.load();
}
