// instance_worker.cpp — the executable of one FixedGSL instance process
// (SAGE_INSTANCE_PROCESS, csrc/fixedgsl.cu): libsagedp runs the serial chain
// over the memfd region whose descriptor it was started with.
#include <cstdlib>

extern "C" int sage_instance_child(int fd);

int main(int argc, char **argv) { return argc < 2 ? 2 : sage_instance_child(std::atoi(argv[1])); }
