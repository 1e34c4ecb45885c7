// Round-trips a matrix file through adpb200_io.hpp (the C++ façade's reader
// and writer of the reference's matrix formats): io_check <in> <out> reads <in> (either
// format) and writes it to <out> (format by extension).
#include <cstdio>
#include <exception>

#include "adpb200_io.hpp"

int main(int argc, char** argv) {
    if (argc != 3) return 2;
    try {
        adpb200::MatrixF64 m = adpb200::read_matrix(argv[1]);
        adpb200::write_matrix(argv[2], m);
        std::printf("%zu %zu\n", m.rows(), m.cols());
    } catch (const std::exception& e) {
        std::fprintf(stderr, "%s\n", e.what());
        return 3;
    }
    return 0;
}
