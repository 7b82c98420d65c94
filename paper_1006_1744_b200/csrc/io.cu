// On-disk matrix and permutation formats (proj/include/f2lin/io.hpp:3-11,
// proj/src/io.cpp), host side of the boundary.
//
//  binary "BMF2": 'B','M','F','2', version 0x01, nrows and ncols as u64 LE, then
//                 nrows * ceil(ncols/64) u64 LE words row-major, padding bits zero;
//  ascii:         "<nrows> <ncols>\n" then nrows lines of ncols characters 0/1.
//
// A binary payload streams straight into HBM: rows are read in chunks into two
// pinned staging buffers and copied with cudaMemcpy2DAsync (file row pitch ->
// 128-B aligned device pitch) on a private stream, so the disk read of chunk c+1
// overlaps the H2D copy of chunk c; stores run the same pipeline in reverse.
// The format validation (magic, version, 2^32 dimension limit, truncation,
// nonzero padding bits, ascii row length / characters / trailing tokens) follows
// io.cpp:45-115 and reports every violation as F2_FORMAT_ERROR (io::FormatError).
// Host byte order is little-endian (x86-64 / aarch64), so words are copied as is.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/f2lin_gpu.h"

namespace f2g {
int set_error(int code, const std::string& msg);
int set_cuda_error(cudaError_t e, const char* what);
}  // namespace f2g

namespace {

using f2g::set_error;

constexpr uint64_t kDimLimit = uint64_t{1} << 32;  // io.cpp:58, :92

size_t chunk_bytes() {
    const char* e = std::getenv("F2_IO_CHUNK_BYTES");
    size_t v = e ? static_cast<size_t>(std::strtoull(e, nullptr, 10)) : 0;
    return v ? v : (size_t{32} << 20);
}

struct File {
    FILE* f = nullptr;
    explicit File(FILE* x) : f(x) {}
    ~File() {
        if (f) std::fclose(f);
    }
};

struct Header {
    uint64_t m = 0, n = 0;
    int fmt = F2_FMT_ASCII;
};

uint64_t le64(const unsigned char* b) {
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(b[i]) << (8 * i);
    return v;
}

// Binary header after the format sniff (io.cpp:45-61)
int read_binary_header(FILE* f, Header& h) {
    unsigned char b[21];
    const size_t got = std::fread(b, 1, 21, f);
    if (got < 4 || std::memcmp(b, "BMF2", 4) != 0) return set_error(F2_FORMAT_ERROR, "bad magic in binary matrix file");
    if (got < 5 || b[4] != 0x01) return set_error(F2_FORMAT_ERROR, "unsupported binary matrix version");
    if (got < 21) return set_error(F2_FORMAT_ERROR, "truncated binary matrix file");
    h.m = le64(b + 5);
    h.n = le64(b + 13);
    h.fmt = F2_FMT_BINARY;
    if (h.m >= kDimLimit || h.n >= kDimLimit) return set_error(F2_FORMAT_ERROR, "matrix dimensions overflow");
    return F2_OK;
}

// ascii header line "<nrows> <ncols>" with nothing after it (io.cpp:82-92)
int parse_ascii_header(const std::string& line, Header& h) {
    std::istringstream hs(line);
    uint64_t m = 0, n = 0;
    if (!(hs >> m >> n)) return set_error(F2_FORMAT_ERROR, "malformed header line");
    std::string rest;
    if (hs >> rest) return set_error(F2_FORMAT_ERROR, "malformed header line");
    if (m >= kDimLimit || n >= kDimLimit) return set_error(F2_FORMAT_ERROR, "matrix dimensions overflow");
    h.m = m;
    h.n = n;
    h.fmt = F2_FMT_ASCII;
    return F2_OK;
}

bool read_line(FILE* f, std::string& out) {
    out.clear();
    int c;
    bool any = false;
    while ((c = std::fgetc(f)) != EOF) {
        any = true;
        if (c == '\n') return true;
        out.push_back(static_cast<char>(c));
    }
    return any;
}

// Sniff + header: an ascii file starts with a digit, the binary magic with 'B'
// (io.cpp:118-126).
int open_and_header(const char* path, File& file, Header& h) {
    if (!path) return set_error(F2_INVALID_ARGUMENT, "path is NULL");
    file.f = std::fopen(path, "rb");
    if (!file.f) return set_error(F2_FORMAT_ERROR, std::string("cannot open for reading: ") + path);
    std::setvbuf(file.f, nullptr, _IOFBF, 1 << 20);
    const int c = std::fgetc(file.f);
    if (c != EOF) std::ungetc(c, file.f);
    if (c == 'B') return read_binary_header(file.f, h);
    std::string line;
    if (!read_line(file.f, line)) return set_error(F2_FORMAT_ERROR, "missing header line");
    return parse_ascii_header(line, h);
}

// Streams the payload in row batches: sink(r0, rows, words, row_words), `words`
// in file packing (row pitch ceil(n/64)).  `stage` gives the buffer for a batch.
using Stage = std::function<uint64_t*(size_t batch_index)>;
using Sink = std::function<int(size_t r0, size_t rows, uint64_t* words, size_t batch_index)>;

int stream_payload(FILE* f, const Header& h, size_t batch_rows, const Stage& stage, const Sink& sink) {
    const size_t nw = (h.n + 63) / 64;
    const unsigned used = static_cast<unsigned>(h.n % 64);
    const uint64_t pad = used ? ~((uint64_t{1} << used) - 1) : 0;
    size_t bi = 0;
    std::string line;
    for (size_t r0 = 0; r0 < h.m; r0 += batch_rows, ++bi) {
        const size_t rows = std::min<size_t>(batch_rows, h.m - r0);
        uint64_t* buf = stage(bi);
        if (h.fmt == F2_FMT_BINARY) {
            const size_t got = nw ? std::fread(buf, 8 * nw, rows, f) : rows;
            for (size_t i = 0; i < got; ++i)
                if (nw && (buf[i * nw + nw - 1] & pad))
                    return set_error(F2_FORMAT_ERROR, "nonzero padding bits in binary matrix file");
            if (got < rows) return set_error(F2_FORMAT_ERROR, "truncated binary matrix file");
        } else {
            std::memset(buf, 0, 8 * nw * rows);
            for (size_t i = 0; i < rows; ++i) {
                if (!read_line(f, line)) return set_error(F2_FORMAT_ERROR, "missing matrix row");
                if (!line.empty() && line.back() == '\r') line.pop_back();
                if (line.size() != h.n) return set_error(F2_FORMAT_ERROR, "matrix row has the wrong length");
                uint64_t* row = buf + i * nw;
                for (size_t j = 0; j < h.n; ++j) {
                    const char ch = line[j];
                    if (ch == '1') row[j >> 6] |= uint64_t{1} << (j & 63);
                    else if (ch != '0')
                        return set_error(F2_FORMAT_ERROR, "matrix row contains characters other than 0/1");
                }
            }
        }
        int rc = sink(r0, rows, buf, bi);
        if (rc) return rc;
    }
    return F2_OK;
}

int write_all(FILE* f, const void* p, size_t bytes) {
    return std::fwrite(p, 1, bytes, f) == bytes ? F2_OK : set_error(F2_FORMAT_ERROR, "write failed");
}

int write_header(FILE* f, uint64_t m, uint64_t n, int fmt) {
    if (fmt == F2_FMT_BINARY) {
        unsigned char b[21] = {'B', 'M', 'F', '2', 0x01};
        for (int i = 0; i < 8; ++i) {
            b[5 + i] = static_cast<unsigned char>(m >> (8 * i));
            b[13 + i] = static_cast<unsigned char>(n >> (8 * i));
        }
        return write_all(f, b, sizeof b);
    }
    std::string s = std::to_string(m) + " " + std::to_string(n) + "\n";
    return write_all(f, s.data(), s.size());
}

// rows of packed words (pitch nw) in the requested format
int write_rows(FILE* f, const uint64_t* w, size_t rows, uint64_t n, int fmt, std::string& line) {
    const size_t nw = (n + 63) / 64;
    if (fmt == F2_FMT_BINARY) return write_all(f, w, 8 * nw * rows);
    line.resize(n + 1);
    line[n] = '\n';
    for (size_t i = 0; i < rows; ++i) {
        const uint64_t* row = w + i * nw;
        for (size_t j = 0; j < n; ++j) line[j] = ((row[j >> 6] >> (j & 63)) & 1) ? '1' : '0';
        int rc = write_all(f, line.data(), line.size());
        if (rc) return rc;
    }
    return F2_OK;
}

int open_for_write(const char* path, File& file, int fmt) {
    if (!path) return set_error(F2_INVALID_ARGUMENT, "path is NULL");
    if (fmt != F2_FMT_ASCII && fmt != F2_FMT_BINARY) return set_error(F2_INVALID_ARGUMENT, "unknown format");
    file.f = std::fopen(path, "wb");
    if (!file.f) return set_error(F2_FORMAT_ERROR, std::string("cannot open for writing: ") + path);
    std::setvbuf(file.f, nullptr, _IOFBF, 1 << 20);
    return F2_OK;
}

int close_written(File& file) {
    FILE* f = file.f;
    file.f = nullptr;
    return std::fclose(f) == 0 ? F2_OK : set_error(F2_FORMAT_ERROR, "write failed");
}

// Two pinned staging buffers + events on a private stream.
struct Pipe {
    cudaStream_t s = nullptr;
    uint64_t* buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    bool used[2] = {false, false};
    ~Pipe() {
        if (s) cudaStreamSynchronize(s);
        for (int i = 0; i < 2; ++i) {
            if (buf[i]) cudaFreeHost(buf[i]);
            if (ev[i]) cudaEventDestroy(ev[i]);
        }
        if (s) cudaStreamDestroy(s);
    }
    int init(size_t bytes) {
        cudaError_t e;
        if ((e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)) != cudaSuccess)
            return f2g::set_cuda_error(e, "io stream");
        for (int i = 0; i < 2; ++i) {
            if ((e = cudaMallocHost(&buf[i], bytes ? bytes : 8)) != cudaSuccess) return f2g::set_cuda_error(e, "io staging");
            if ((e = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming)) != cudaSuccess)
                return f2g::set_cuda_error(e, "io event");
        }
        return F2_OK;
    }
    uint64_t* wait(size_t bi) {  // buffer bi%2, once its previous copy is done
        const int b = static_cast<int>(bi & 1);
        if (used[b]) cudaEventSynchronize(ev[b]);
        return buf[b];
    }
    int issued(size_t bi) {
        const int b = static_cast<int>(bi & 1);
        used[b] = true;
        cudaError_t e = cudaEventRecord(ev[b], s);
        return e == cudaSuccess ? F2_OK : f2g::set_cuda_error(e, "io event record");
    }
};

}  // namespace

extern "C" {

int f2_io_probe(const char* path, uint64_t* nrows, uint64_t* ncols, int* format) {
    File file(nullptr);
    Header h;
    int rc = open_and_header(path, file, h);
    if (rc) return rc;
    if (nrows) *nrows = h.m;
    if (ncols) *ncols = h.n;
    if (format) *format = h.fmt;
    return F2_OK;
}

int f2_io_read_host(const char* path, uint64_t* words, size_t stride_words, uint64_t nrows, uint64_t ncols) {
    File file(nullptr);
    Header h;
    int rc = open_and_header(path, file, h);
    if (rc) return rc;
    if (h.m != nrows || h.n != ncols) return set_error(F2_INVALID_ARGUMENT, "file dimensions differ from the buffer's");
    const size_t nw = (h.n + 63) / 64;
    if (stride_words < nw || (!words && h.m && nw)) return set_error(F2_INVALID_ARGUMENT, "bad host buffer");
    std::vector<uint64_t> tmp(nw ? nw : 1);
    return stream_payload(
        file.f, h, 1, [&](size_t) { return tmp.data(); },
        [&](size_t r0, size_t, uint64_t* w, size_t) {
            if (nw) std::memcpy(words + r0 * stride_words, w, 8 * nw);
            return F2_OK;
        });
}

int f2_io_write_host(const char* path, const uint64_t* words, size_t stride_words, uint64_t nrows, uint64_t ncols,
                     int format) {
    const size_t nw = (ncols + 63) / 64;
    if (stride_words < nw || (!words && nrows && nw)) return set_error(F2_INVALID_ARGUMENT, "bad host buffer");
    File file(nullptr);
    int rc = open_for_write(path, file, format);
    if (rc || (rc = write_header(file.f, nrows, ncols, format))) return rc;
    std::string line;
    std::vector<uint64_t> row(nw ? nw : 1);
    const unsigned used = static_cast<unsigned>(ncols % 64);
    for (uint64_t i = 0; i < nrows; ++i) {
        if (nw) std::memcpy(row.data(), words + i * stride_words, 8 * nw);
        if (used) row[nw - 1] &= (uint64_t{1} << used) - 1;  // BitMatrix padding is zero
        if ((rc = write_rows(file.f, row.data(), 1, ncols, format, line))) return rc;
    }
    return close_written(file);
}

// io::read_matrix(path, &detected) -> a new HBM-resident matrix
int f2_matrix_load(const char* path, f2_matrix** out, int* detected) {
    if (!out) return set_error(F2_INVALID_ARGUMENT, "out is NULL");
    File file(nullptr);
    Header h;
    int rc = open_and_header(path, file, h);
    if (rc) return rc;
    f2_matrix* a = nullptr;
    if ((rc = f2_matrix_create(h.m, h.n, &a))) return rc;
    const size_t nw = (h.n + 63) / 64, dpitch = 8 * f2_matrix_stride(a);
    uint64_t* dev = f2_matrix_device_ptr(a);
    const size_t batch = std::max<size_t>(1, chunk_bytes() / std::max<size_t>(8 * nw, 1));
    {
        Pipe pipe;
        if ((rc = pipe.init(8 * nw * std::min<size_t>(batch, std::max<uint64_t>(h.m, 1))))) {
            f2_matrix_destroy(a);
            return rc;
        }
        rc = stream_payload(
            file.f, h, batch, [&](size_t bi) { return pipe.wait(bi); },
            [&](size_t r0, size_t rows, uint64_t* w, size_t bi) {
                if (nw) {
                    cudaError_t e = cudaMemcpy2DAsync(reinterpret_cast<char*>(dev) + r0 * dpitch, dpitch, w, 8 * nw,
                                                      8 * nw, rows, cudaMemcpyHostToDevice, pipe.s);
                    if (e != cudaSuccess) return f2g::set_cuda_error(e, "io upload");
                }
                return pipe.issued(bi);
            });
        cudaError_t e = cudaStreamSynchronize(pipe.s);
        if (!rc && e != cudaSuccess) rc = f2g::set_cuda_error(e, "io upload");
    }
    if (rc) {
        f2_matrix_destroy(a);
        return rc;
    }
    if (detected) *detected = h.fmt;
    *out = a;
    return F2_OK;
}

// io::write_matrix(path, a, fmt) from HBM
int f2_matrix_store(const f2_matrix* a, const char* path, int format) {
    if (!a) return set_error(F2_INVALID_ARGUMENT, "null argument");
    const uint64_t m = f2_matrix_nrows(a), n = f2_matrix_ncols(a);
    const size_t nw = (n + 63) / 64, spitch = 8 * f2_matrix_stride(a);
    const uint64_t* dev = f2_matrix_device_ptr(const_cast<f2_matrix*>(a));
    File file(nullptr);
    int rc = open_for_write(path, file, format);
    if (rc || (rc = write_header(file.f, m, n, format))) return rc;
    std::string empty;
    if (m && !nw && (rc = write_rows(file.f, nullptr, m, n, format, empty))) return rc;  // zero-width rows
    if (m && nw) {
        const size_t batch = std::max<size_t>(1, chunk_bytes() / (8 * nw));
        Pipe pipe;
        if ((rc = pipe.init(8 * nw * std::min<size_t>(batch, m)))) return rc;
        std::string line;
        const size_t nb = (m + batch - 1) / batch;
        auto issue = [&](size_t bi) -> int {
            const size_t r0 = bi * batch, rows = std::min<size_t>(batch, m - r0);
            cudaError_t e = cudaMemcpy2DAsync(pipe.buf[bi & 1], 8 * nw, reinterpret_cast<const char*>(dev) + r0 * spitch,
                                              spitch, 8 * nw, rows, cudaMemcpyDeviceToHost, pipe.s);
            if (e != cudaSuccess) return f2g::set_cuda_error(e, "io download");
            return pipe.issued(bi);
        };
        if ((rc = issue(0))) return rc;
        for (size_t bi = 0; bi < nb; ++bi) {
            cudaEventSynchronize(pipe.ev[bi & 1]);
            if (bi + 1 < nb && (rc = issue(bi + 1))) return rc;  // next copy overlaps this write
            const size_t rows = std::min<size_t>(batch, m - bi * batch);
            if ((rc = write_rows(file.f, pipe.buf[bi & 1], rows, n, format, line))) return rc;
        }
    }
    return close_written(file);
}

// io::write_permutation: one line of space-separated entries (io.cpp:135-142)
int f2_write_permutation(const char* path, const uint64_t* p, size_t len) {
    if (!p && len) return set_error(F2_INVALID_ARGUMENT, "null argument");
    File file(nullptr);
    if (!path) return set_error(F2_INVALID_ARGUMENT, "path is NULL");
    file.f = std::fopen(path, "w");
    if (!file.f) return set_error(F2_FORMAT_ERROR, std::string("cannot open for writing: ") + path);
    std::string s;
    for (size_t i = 0; i < len; ++i) {
        if (i) s.push_back(' ');
        s += std::to_string(p[i]);
    }
    s.push_back('\n');
    int rc = write_all(file.f, s.data(), s.size());
    if (rc) return rc;
    return close_written(file);
}

// io::read_permutation: entries of the first line until the first non-number
// (io.cpp:150-160).  *len is always set; entries are copied when len <= cap.
int f2_read_permutation(const char* path, uint64_t* p, size_t cap, size_t* len) {
    if (!path || !len) return set_error(F2_INVALID_ARGUMENT, "null argument");
    std::ifstream in(path);
    if (!in) return set_error(F2_FORMAT_ERROR, std::string("cannot open for reading: ") + path);
    std::string line;
    if (!std::getline(in, line)) return set_error(F2_FORMAT_ERROR, "missing permutation line");
    std::istringstream ls(line);
    std::vector<uint64_t> v;
    unsigned long long x;
    while (ls >> x) v.push_back(x);
    *len = v.size();
    if (v.size() > cap) return p ? set_error(F2_INVALID_ARGUMENT, "permutation buffer too small") : F2_OK;
    if (!v.empty()) std::memcpy(p, v.data(), 8 * v.size());
    return F2_OK;
}

}  // extern "C"
