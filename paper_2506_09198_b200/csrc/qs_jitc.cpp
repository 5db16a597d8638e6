// qs_jitc.cpp — the background compiler process of the JIT tile executor (jit_tile.cu): compiles each
// source file named on the command line into the on-disk cubin cache (NVRTC, sm_100a) and deletes it.
// Runs detached from the application, so a compilation still in flight when the application exits
// cannot crash or stall the application's exit.
extern "C" int qs_jit_compile_file(const char *path);

int main(int argc, char **argv) {
    int rc = 0;
    for (int i = 1; i < argc; ++i) rc |= qs_jit_compile_file(argv[i]);
    return rc;
}
