// fp8t_io.cu -- host-side FP8T container I/O (tensor_io.cpp:47-187), the format
// the reference uses for golden vectors and checkpoints. No device code: the
// callers move tensors between HBM and these host buffers.
#include <cstdint>
#include <cstdio>
#include <exception>
#include <cstring>
#include <string>
#include <vector>

#include "kernels.cuh"

namespace fp8b {
void set_error(const std::string& msg);
}

namespace {

constexpr unsigned char kMagic[4] = {'F', 'P', '8', 'T'};
constexpr unsigned char kVersion = 1;

struct File {
    std::FILE* f = nullptr;
    File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
    ~File() {
        if (f) std::fclose(f);
    }
};

int io_fail(const std::string& msg) {
    fp8b::set_error(msg);
    return FP8B_EIO;
}

size_t elem_bytes(int dtype) { return dtype == FP8B_FP8T_F32 ? 4 : dtype == FP8B_FP8T_FP8 ? 1 : 2; }

struct Header {
    int dtype = 0, mode = 0;
    std::vector<int64_t> dims;
};

// read_header (tensor_io.cpp:64-90), same checks and messages
int read_header(std::FILE* f, const std::string& path, Header& h) {
    unsigned char magic[4];
    if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, kMagic, 4) != 0)
        return io_fail(path + ": not an FP8T tensor file (bad magic)");
    unsigned char head[4], reserved[8];
    if (std::fread(head, 1, 4, f) != 4 || std::fread(reserved, 1, 8, f) != 8)
        return io_fail(path + ": truncated FP8T header");
    if (head[0] != kVersion)
        return io_fail(path + ": unsupported FP8T version " + std::to_string(head[0]));
    if (head[1] > 2) return io_fail(path + ": unknown FP8T dtype tag " + std::to_string(head[1]));
    h.dtype = head[1];
    h.mode = head[3];
    h.dims.resize(head[2]);
    for (auto& d : h.dims) {
        unsigned char b[8];
        if (std::fread(b, 1, 8, f) != 8) return io_fail(path + ": truncated FP8T dimension list");
        uint64_t v = 0;
        for (int i = 0; i < 8; ++i) v = (v << 8) | b[i];
        d = (int64_t)v;
        // shape_numel (tensor.cpp:9-16) throws invalid_argument here
        if (d < 0) return io_fail("negative dimension");
    }
    int64_t n = 1;
    for (int64_t d : h.dims) {
        if (d != 0 && n > INT64_MAX / 4 / d) return io_fail(path + ": dimension product overflows");
        n *= d;
    }
    return FP8B_OK;
}

// Dims are non-negative and their product (times 4 bytes) fits int64: checked
// by read_header / fp8b_fp8t_save before this is called.
int64_t numel(const std::vector<int64_t>& dims) {
    int64_t n = 1;
    for (int64_t d : dims) n *= d;
    return n;
}

}  // namespace

extern "C" {

int fp8b_fp8t_save(const char* path, int32_t dtype, int32_t mode_tag, int32_t rank,
                   const int64_t* dims, const void* data) {
    if (!path) return io_fail("fp8t_save: null path");
    if (dtype < 0 || dtype > 2) return io_fail(std::string(path) + ": unknown FP8T dtype tag");
    if (rank < 0 || rank > FP8B_FP8T_MAX_RANK || (rank > 0 && !dims))
        return io_fail(std::string(path) + ": bad rank");
    if (mode_tag < 0 || mode_tag > 3) return io_fail(std::string(path) + ": unknown rounding mode tag");
    std::vector<int64_t> d(dims, dims + rank);
    int64_t prod = 1;
    for (int64_t v : d) {
        if (v < 0) return io_fail(std::string(path) + ": negative dimension");
        if (v != 0 && prod > INT64_MAX / 4 / v)
            return io_fail(std::string(path) + ": dimension product overflows");
        prod *= v;
    }
    const int64_t n = numel(d);
    if (n > 0 && !data) return io_fail(std::string(path) + ": null payload");
    File out(path, "wb");
    if (!out.f) return io_fail(std::string(path) + ": cannot open for writing");
    // write_header (tensor_io.cpp:47-57)
    std::vector<unsigned char> buf;
    buf.insert(buf.end(), kMagic, kMagic + 4);
    buf.push_back(kVersion);
    buf.push_back((unsigned char)dtype);
    buf.push_back((unsigned char)rank);
    buf.push_back((unsigned char)(dtype == FP8B_FP8T_F32 ? 0 : mode_tag));
    buf.insert(buf.end(), 8, 0);
    for (int64_t v : d)
        for (int i = 0; i < 8; ++i) buf.push_back((unsigned char)((uint64_t)v >> (56 - 8 * i)));
    const size_t eb = elem_bytes(dtype);
    const size_t hdr = buf.size();
    try {
        buf.resize(hdr + (size_t)n * eb);
    } catch (const std::exception&) {  // never let an exception cross the C ABI
        return io_fail(std::string(path) + ": cannot allocate the payload buffer");
    }
    unsigned char* p = buf.data() + hdr;
    if (dtype == FP8B_FP8T_FP8) {
        std::memcpy(p, data, (size_t)n);
    } else if (dtype == FP8B_FP8T_FP16) {
        const uint16_t* s = static_cast<const uint16_t*>(data);
        for (int64_t i = 0; i < n; ++i) {
            p[2 * i] = (unsigned char)(s[i] >> 8);
            p[2 * i + 1] = (unsigned char)(s[i] & 0xFF);
        }
    } else {
        const uint32_t* s = static_cast<const uint32_t*>(data);
        for (int64_t i = 0; i < n; ++i) {
            p[4 * i] = (unsigned char)(s[i] >> 24);
            p[4 * i + 1] = (unsigned char)(s[i] >> 16);
            p[4 * i + 2] = (unsigned char)(s[i] >> 8);
            p[4 * i + 3] = (unsigned char)s[i];
        }
    }
    if (std::fwrite(buf.data(), 1, buf.size(), out.f) != buf.size())
        return io_fail(std::string(path) + ": write failed");
    return FP8B_OK;
}

int fp8b_fp8t_peek(const char* path, int32_t* dtype, int32_t* mode_tag, int32_t* rank,
                   int64_t* dims, int32_t max_rank) {
    if (!path) return io_fail("fp8t_peek: null path");
    File in(path, "rb");
    if (!in.f) return io_fail(std::string(path) + ": cannot open for reading");
    Header h;
    const int rc = read_header(in.f, path, h);
    if (rc) return rc;
    if (dtype) *dtype = h.dtype;
    if (mode_tag) *mode_tag = h.mode;
    if (rank) *rank = (int32_t)h.dims.size();
    if (dims)
        for (size_t i = 0; i < h.dims.size() && (int32_t)i < max_rank; ++i) dims[i] = h.dims[i];
    return FP8B_OK;
}

int fp8b_fp8t_load(const char* path, int32_t expect_dtype, void* data, int64_t capacity) {
    if (!path) return io_fail("fp8t_load: null path");
    File in(path, "rb");
    if (!in.f) return io_fail(std::string(path) + ": cannot open for reading");
    Header h;
    const int rc = read_header(in.f, path, h);
    if (rc) return rc;
    if (expect_dtype == FP8B_FP8T_F32 && h.dtype != FP8B_FP8T_F32)
        return io_fail(std::string(path) + ": expected FP32 payload (dtype 0)");
    if (expect_dtype != FP8B_FP8T_F32 && h.dtype == FP8B_FP8T_F32)
        return io_fail(std::string(path) + ": holds FP32 data, not codes");
    if (h.dtype != FP8B_FP8T_F32 && h.mode > 3)
        return io_fail(std::string(path) + ": unknown rounding mode tag");
    const int64_t n = numel(h.dims);
    if (n > capacity) return io_fail(std::string(path) + ": payload larger than the buffer");
    const size_t eb = elem_bytes(h.dtype);
    std::vector<unsigned char> buf;
    try {
        buf.resize((size_t)n * eb);
    } catch (const std::exception&) {  // never let an exception cross the C ABI
        return io_fail(std::string(path) + ": cannot allocate the payload buffer");
    }
    if (n > 0 && std::fread(buf.data(), 1, buf.size(), in.f) != buf.size())
        return io_fail(std::string(path) +
                       (h.dtype == FP8B_FP8T_F32 ? ": truncated FP32 payload" : ": truncated code payload"));
    const unsigned char* p = buf.data();
    if (h.dtype == FP8B_FP8T_FP8) {
        std::memcpy(data, p, (size_t)n);
    } else if (h.dtype == FP8B_FP8T_FP16) {
        uint16_t* d = static_cast<uint16_t*>(data);
        for (int64_t i = 0; i < n; ++i) d[i] = (uint16_t)((p[2 * i] << 8) | p[2 * i + 1]);
    } else {
        uint32_t* d = static_cast<uint32_t*>(data);
        for (int64_t i = 0; i < n; ++i)
            d[i] = ((uint32_t)p[4 * i] << 24) | ((uint32_t)p[4 * i + 1] << 16) |
                   ((uint32_t)p[4 * i + 2] << 8) | p[4 * i + 3];
    }
    return FP8B_OK;
}

}  // extern "C"
