// oracle/ref_io_tool.cpp -- TEST INFRASTRUCTURE ONLY: a command-line view of
// the UNMODIFIED reference's matrix IO (io.cpp), run as a subprocess by the
// tests (the reference's formatted MatrixMarket writer crashes inside a
// python process that has numpy's bundled libquadmath loaded; standalone it
// is fine).  Usage:
//   ref_io_tool convert <in_fmt> <in_path> <out_fmt> <out_path>
// reads with read_matrix_file(in_path, in_fmt), writes with
// write_matrix_file(out_path, ., out_fmt).  Exit 0, or 1 with the message.
#include <cstdio>
#include <cstring>
#include <exception>

#include "taskeig/io.hpp"

int main(int argc, char** argv) {
    if (argc != 6 || std::strcmp(argv[1], "convert") != 0) {
        std::fprintf(stderr, "usage: ref_io_tool convert <in_fmt> <in> <out_fmt> <out>\n");
        return 64;
    }
    try {
        auto m = taskeig::read_matrix_file(argv[3], argv[2]);
        taskeig::write_matrix_file(argv[5], m, argv[4]);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "%s\n", e.what());
        return 1;
    }
    return 0;
}
