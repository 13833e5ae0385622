// io.cpp -- matrix files of the reference's formats (
// reference io.hpp / io.cpp:37-121), host side of the CLI:
//   TEIG          "TEIG" | uint32 version 1 | uint64 rows | uint64 cols |
//                 rows*cols float64, ROW-major, native byte order
//   MatrixMarket  "%%MatrixMarket matrix array real general", "rows cols",
//                 then the entries column by column, one per line, printed
//                 with 17 significant digits
// Byte-compatible with the reference in both directions (tests/test_io.py).
// The in-memory interchange is row-major (the reference's DenseBuffer).
#include <algorithm>
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/taskeig_b200.h"

namespace teig {
int set_error(int code, const std::string& msg);
}

using namespace teig;

namespace {

int fmt_of(const char* format) {
    if (!format) return -1;
    if (!std::strcmp(format, "teig")) return 0;
    if (!std::strcmp(format, "matrixmarket")) return 1;
    return -1;
}

void write_teig(const char* path, uint64_t rows, uint64_t cols, const double* a) {
    std::ofstream os(path, std::ios::binary);
    if (!os) throw std::runtime_error(std::string("cannot open for writing: ") + path);
    const uint32_t version = 1;
    os.write("TEIG", 4);
    os.write(reinterpret_cast<const char*>(&version), sizeof version);
    os.write(reinterpret_cast<const char*>(&rows), sizeof rows);
    os.write(reinterpret_cast<const char*>(&cols), sizeof cols);
    os.write(reinterpret_cast<const char*>(a), (std::streamsize)(rows * cols * sizeof(double)));
    if (!os) throw std::runtime_error(std::string("short write: ") + path);
}

void read_teig(const char* path, uint64_t* rows, uint64_t* cols, double* a, uint64_t cap) {
    std::ifstream is(path, std::ios::binary);
    if (!is) throw std::runtime_error(std::string("cannot open: ") + path);
    char magic[4];
    is.read(magic, 4);
    if (!is || std::memcmp(magic, "TEIG", 4) != 0) throw std::runtime_error(std::string("not a TEIG file: ") + path);
    uint32_t version = 0;
    is.read(reinterpret_cast<char*>(&version), sizeof version);
    if (!is) throw std::runtime_error("teig: truncated file");
    if (version != 1) throw std::runtime_error("unsupported TEIG version");
    is.read(reinterpret_cast<char*>(rows), sizeof *rows);
    is.read(reinterpret_cast<char*>(cols), sizeof *cols);
    if (!is) throw std::runtime_error("teig: truncated file");
    if (!a) return;  // header only
    if (*rows * *cols > cap) throw std::length_error("teig: buffer too small");
    is.read(reinterpret_cast<char*>(a), (std::streamsize)(*rows * *cols * sizeof(double)));
    if (!is) throw std::runtime_error("teig: truncated data section");
}

void write_mm(const char* path, uint64_t rows, uint64_t cols, const double* a) {
    std::ofstream os(path);
    if (!os) throw std::runtime_error(std::string("cannot open for writing: ") + path);
    os << "%%MatrixMarket matrix array real general\n" << rows << " " << cols << "\n";
    os.precision(17);
    for (uint64_t j = 0; j < cols; ++j)
        for (uint64_t i = 0; i < rows; ++i) os << a[i * cols + j] << "\n";
    if (!os) throw std::runtime_error(std::string("short write: ") + path);
}

void read_mm(const char* path, uint64_t* rows, uint64_t* cols, double* a, uint64_t cap) {
    std::ifstream is(path);
    if (!is) throw std::runtime_error(std::string("cannot open: ") + path);
    std::string line;
    if (!std::getline(is, line)) throw std::runtime_error(std::string("empty file: ") + path);
    if (line.rfind("%%MatrixMarket", 0) != 0) throw std::runtime_error(std::string("not a MatrixMarket file: ") + path);
    std::istringstream hs(line);
    std::string mm, obj, fmt, field, sym;
    hs >> mm >> obj >> fmt >> field >> sym;
    if (obj != "matrix" || fmt != "array" || field != "real" || sym != "general")
        throw std::runtime_error("unsupported MatrixMarket flavor: " + line);
    while (std::getline(is, line))
        if (!line.empty() && line[0] != '%') break;
    std::istringstream ds(line);
    if (!(ds >> *rows >> *cols)) throw std::runtime_error(std::string("bad size line: ") + path);
    if (!a) return;
    if (*rows * *cols > cap) throw std::length_error("matrixmarket: buffer too small");
    for (uint64_t j = 0; j < *cols; ++j)
        for (uint64_t i = 0; i < *rows; ++i)
            if (!(is >> a[i * *cols + j]))
                throw std::runtime_error(std::string("truncated MatrixMarket body: ") + path);
}

}  // namespace

extern "C" {

int teig_write_matrix_file(const char* path, const char* format, int64_t rows, int64_t cols, const double* a_rm) {
    const int f = fmt_of(format);
    if (f < 0) return set_error(-2, std::string("unknown matrix format: ") + (format ? format : "(null)"));
    if (!path) return set_error(-1, "path is null");
    if (rows < 0 || cols < 0 || (rows * cols > 0 && !a_rm)) return set_error(-3, "bad matrix");
    try {
        if (f == 0) write_teig(path, (uint64_t)rows, (uint64_t)cols, a_rm);
        else write_mm(path, (uint64_t)rows, (uint64_t)cols, a_rm);
    } catch (const std::exception& e) {
        return set_error(TEIG_ERR_IO, e.what());
    }
    return 0;
}

int teig_read_matrix_file(const char* path, const char* format, int64_t* rows, int64_t* cols, double* a_rm,
                          int64_t cap) {
    const int f = fmt_of(format);
    if (f < 0) return set_error(-2, std::string("unknown matrix format: ") + (format ? format : "(null)"));
    if (!path || !rows || !cols) return set_error(-1, "null argument");
    uint64_t r = 0, c = 0;
    try {
        if (f == 0) read_teig(path, &r, &c, a_rm, (uint64_t)std::max<int64_t>(cap, 0));
        else read_mm(path, &r, &c, a_rm, (uint64_t)std::max<int64_t>(cap, 0));
    } catch (const std::exception& e) {
        return set_error(TEIG_ERR_IO, e.what());
    }
    *rows = (int64_t)r;
    *cols = (int64_t)c;
    return 0;
}

}  // extern "C"
