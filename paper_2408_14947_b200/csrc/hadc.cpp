// hadc.cpp — the reference's HADC cube / mask container (SPEC.md:576-598,
// [MODULE] io: CubeFileHeader, read_cube / write_cube, read_mask / write_mask)
// with a pinned, double-buffered path straight into device memory
// (SURVEY.md §8 f4), so a line-scan run can stream a cube file into the
// engine without a pageable copy.
//
// Byte layout (little-endian; the SPEC names the fields but not their widths,
// pinned here and in DESIGN.md):
//   0  "HADC"            4 bytes
//   4  version  u16      = 1
//   6  lines    u32      >= 1
//  10  pixels   u32      >= 1
//  14  bands    u32      >= 1
//  18  dtype    u8       1 = float32 LE, 2 = u8 (masks: values 0/1, bands = 1)
//  19  layout   u8       1 = line-major [line][pixel][band]
//  20  name_len u16, then name_len bytes of UTF-8 name
//  22+name_len  payload, lines * pixels * bands * sizeof(dtype) bytes, nothing after it
// A malformed or truncated file is had::FormatError (errors.hpp:67-75, kind
// data): ERX_ERR_DATA with "<what> at offset <n>" in the message (SPEC.md:585
// "format error with offset").  Only failing to open or read the file is an
// IoError (ERX_ERR_IO, errors.hpp:77-79).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/erx_b200.h"

struct erx_hadc {
    FILE* f = nullptr;
    erx_hadc_info info{};
    uint64_t payload_off = 0;
    std::string err;
    void* stage[2] = {nullptr, nullptr};
    size_t stage_bytes = 0;
    cudaEvent_t done[2] = {nullptr, nullptr};
};

namespace {

thread_local std::string g_open_err;

constexpr uint32_t kHeaderFixed = 22;

size_t elem_size(uint8_t dtype) { return dtype == 1 ? 4 : (dtype == 2 ? 1 : 0); }

template <typename T>
T rd(const unsigned char* p) {
    T v;
    std::memcpy(&v, p, sizeof(T));
    return v;  // the container is little-endian, as is every CUDA host
}

int open_impl(const char* path, erx_hadc* h) {
    char msg[256];
    h->f = std::fopen(path, "rb");
    if (!h->f) {
        h->err = std::string("cannot open ") + path;
        return ERX_ERR_IO;
    }
    unsigned char hdr[kHeaderFixed];
    const size_t got = std::fread(hdr, 1, kHeaderFixed, h->f);
    if (got < kHeaderFixed) {
        std::snprintf(msg, sizeof msg, "%s: truncated header at offset %zu (need %u bytes)", path, got, kHeaderFixed);
        h->err = msg;
        return ERX_ERR_DATA;
    }
    if (std::memcmp(hdr, "HADC", 4) != 0) {
        h->err = std::string(path) + ": bad magic at offset 0";
        return ERX_ERR_DATA;
    }
    erx_hadc_info& in = h->info;
    in.version = rd<uint16_t>(hdr + 4);
    in.lines = rd<uint32_t>(hdr + 6);
    in.pixels = rd<uint32_t>(hdr + 10);
    in.bands = rd<uint32_t>(hdr + 14);
    in.dtype = hdr[18];
    in.layout = hdr[19];
    const uint16_t nlen = rd<uint16_t>(hdr + 20);
    auto bad = [&](const char* what, int off) {
        std::snprintf(msg, sizeof msg, "%s: %s at offset %d", path, what, off);
        h->err = msg;
        return ERX_ERR_DATA;
    };
    if (in.version != 1) return bad("unsupported version", 4);
    if (in.lines == 0) return bad("lines = 0", 6);
    if (in.pixels == 0) return bad("pixels = 0", 10);
    if (in.bands == 0) return bad("bands = 0", 14);
    if (!elem_size(in.dtype)) return bad("unsupported dtype", 18);
    if (in.layout != 1) return bad("unsupported layout", 19);
    std::vector<char> name(nlen);
    if (nlen && std::fread(name.data(), 1, nlen, h->f) != nlen) return bad("truncated name", int(kHeaderFixed));
    in.name_len = nlen;
    std::memset(in.name, 0, sizeof in.name);
    std::memcpy(in.name, name.data(), std::min<size_t>(nlen, sizeof in.name - 1));
    h->payload_off = kHeaderFixed + nlen;
    uint64_t payload = 0;
    if (__builtin_mul_overflow(uint64_t(in.lines), uint64_t(in.pixels), &payload) ||
        __builtin_mul_overflow(payload, uint64_t(in.bands), &payload) ||
        __builtin_mul_overflow(payload, uint64_t(elem_size(in.dtype)), &payload) ||
        payload > (uint64_t(1) << 62))
        return bad("declared payload size overflows", 6);
    std::fseek(h->f, 0, SEEK_END);
    const uint64_t size = uint64_t(std::ftell(h->f));
    if (size != h->payload_off + payload) {
        std::snprintf(msg, sizeof msg, "%s: payload length mismatch at offset %llu: %llu bytes, header declares %llu",
                      path, (unsigned long long)h->payload_off, (unsigned long long)(size - h->payload_off),
                      (unsigned long long)payload);
        h->err = msg;
        return ERX_ERR_DATA;
    }
    return ERX_OK;
}

int read_host(erx_hadc* h, uint32_t first, uint32_t n, void* dst) {
    const erx_hadc_info& in = h->info;
    if (uint64_t(first) + n > in.lines) {
        h->err = "line range past the end of the cube";
        return ERX_ERR_CONFIG;
    }
    const uint64_t line_bytes = uint64_t(in.pixels) * in.bands * elem_size(in.dtype);
    const uint64_t off = h->payload_off + first * line_bytes;
    if (std::fseek(h->f, long(off), SEEK_SET) != 0 ||
        std::fread(dst, 1, size_t(n * line_bytes), h->f) != size_t(n * line_bytes)) {
        char msg[128];
        std::snprintf(msg, sizeof msg, "short read at offset %llu", (unsigned long long)off);
        h->err = msg;
        return ERX_ERR_IO;
    }
    if (in.dtype == 2) {  // masks: 0 / 1 only ("mask value 2 on read -> validation error")
        const unsigned char* p = static_cast<const unsigned char*>(dst);
        for (uint64_t i = 0; i < n * line_bytes; ++i)
            if (p[i] > 1) {
                char msg[128];
                std::snprintf(msg, sizeof msg, "mask value %u at offset %llu", unsigned(p[i]),
                              (unsigned long long)(off + i));
                h->err = msg;
                return ERX_ERR_DATA;
            }
    }
    return ERX_OK;
}

}  // namespace

extern "C" {

int erx_hadc_open(const char* path, erx_hadc** out, erx_hadc_info* info) {
    if (!path || !out) return ERX_ERR_CONFIG;
    *out = nullptr;
    erx_hadc* h = new erx_hadc();
    const int st = open_impl(path, h);
    if (st != ERX_OK) {
        g_open_err = h->err;
        erx_hadc_close(h);
        return st;
    }
    if (info) *info = h->info;
    *out = h;
    return ERX_OK;
}

const char* erx_hadc_last_error(const erx_hadc* h) { return h ? h->err.c_str() : g_open_err.c_str(); }

int erx_hadc_read(erx_hadc* h, uint32_t first_line, uint32_t n_lines, void* dst) {
    if (!h || (n_lines && !dst)) return ERX_ERR_CONFIG;
    return read_host(h, first_line, n_lines, dst);
}

int erx_hadc_read_device(erx_hadc* h, uint32_t first_line, uint32_t n_lines, void* d_dst, void* stream) {
    if (!h || (n_lines && !d_dst)) return ERX_ERR_CONFIG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const erx_hadc_info& in = h->info;
    if (uint64_t(first_line) + n_lines > in.lines) {
        h->err = "line range past the end of the cube";
        return ERX_ERR_CONFIG;
    }
    const uint64_t line_bytes = uint64_t(in.pixels) * in.bands * elem_size(in.dtype);
    // two pinned stages of ~16 MB (whole lines): the file read of chunk c + 1 overlaps the H2D copy of c
    const uint32_t per = uint32_t(std::max<uint64_t>(1, (uint64_t(16) << 20) / line_bytes));
    const size_t need = size_t(per * line_bytes);
    if (h->stage_bytes < need) {
        for (int b = 0; b < 2; ++b) {
            if (h->stage[b]) cudaFreeHost(h->stage[b]);
            h->stage[b] = nullptr;
            if (cudaMallocHost(&h->stage[b], need) != cudaSuccess) {
                h->err = "pinned staging allocation failed";
                return ERX_ERR_DEVICE;
            }
            if (!h->done[b] && cudaEventCreateWithFlags(&h->done[b], cudaEventDisableTiming) != cudaSuccess)
                return ERX_ERR_DEVICE;
        }
        h->stage_bytes = need;
    }
    bool used[2] = {false, false};
    int b = 0;
    for (uint32_t c = 0; c < n_lines; c += per, b ^= 1) {
        const uint32_t m = std::min(per, n_lines - c);
        if (used[b] && cudaEventSynchronize(h->done[b]) != cudaSuccess) return ERX_ERR_DEVICE;
        const int rs = read_host(h, first_line + c, m, h->stage[b]);
        if (rs != ERX_OK) {
            cudaStreamSynchronize(st);
            return rs;
        }
        if (cudaMemcpyAsync(static_cast<char*>(d_dst) + size_t(c) * line_bytes, h->stage[b], size_t(m * line_bytes),
                            cudaMemcpyHostToDevice, st) != cudaSuccess ||
            cudaEventRecord(h->done[b], st) != cudaSuccess)
            return ERX_ERR_DEVICE;
        used[b] = true;
    }
    return cudaStreamSynchronize(st) == cudaSuccess ? ERX_OK : ERX_ERR_DEVICE;
}

void erx_hadc_close(erx_hadc* h) {
    if (!h) return;
    if (h->f) std::fclose(h->f);
    for (int b = 0; b < 2; ++b) {
        if (h->stage[b]) cudaFreeHost(h->stage[b]);
        if (h->done[b]) cudaEventDestroy(h->done[b]);
    }
    delete h;
}

int erx_hadc_write(const char* path, const char* name, uint32_t lines, uint32_t pixels, uint32_t bands,
                   int dtype, const void* data) {
    if (!path || !data || !elem_size(uint8_t(dtype))) return ERX_ERR_CONFIG;
    if (lines == 0 || pixels == 0 || bands == 0) return ERX_ERR_CONFIG;  // SPEC.md:589 "lines=0 -> validation error"
    const uint64_t payload = uint64_t(lines) * pixels * bands * elem_size(uint8_t(dtype));
    if (dtype == 2)
        for (uint64_t i = 0; i < payload; ++i)
            if (static_cast<const unsigned char*>(data)[i] > 1) return ERX_ERR_DATA;
    const size_t nlen = name ? std::strlen(name) : 0;
    if (nlen > 0xFFFF) return ERX_ERR_CONFIG;
    unsigned char hdr[kHeaderFixed];
    std::memcpy(hdr, "HADC", 4);
    const uint16_t ver = 1, nl = uint16_t(nlen);
    std::memcpy(hdr + 4, &ver, 2);
    std::memcpy(hdr + 6, &lines, 4);
    std::memcpy(hdr + 10, &pixels, 4);
    std::memcpy(hdr + 14, &bands, 4);
    hdr[18] = uint8_t(dtype);
    hdr[19] = 1;
    std::memcpy(hdr + 20, &nl, 2);
    FILE* f = std::fopen(path, "wb");
    if (!f) return ERX_ERR_IO;
    bool ok = std::fwrite(hdr, 1, kHeaderFixed, f) == kHeaderFixed;
    ok = ok && (nlen == 0 || std::fwrite(name, 1, nlen, f) == nlen);
    ok = ok && std::fwrite(data, 1, size_t(payload), f) == size_t(payload);
    ok = (std::fclose(f) == 0) && ok;
    return ok ? ERX_OK : ERX_ERR_IO;
}

}  // extern "C"
