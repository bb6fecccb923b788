// formats.cpp — the on-disk formats around the path:
//   * PKVT trace: cached (X, Y) score pairs,
//     magic "PKVT", u32 version, u64 header length, textual key=value header
//     (geometry L_s,H_s,L_l,H_l,N,B, dtype, sample count, free metadata),
//     payload per sample X [B,L_s,H_s,N] then Y [B,L_l,H_l,N], little-endian
//     fp32. read(write(t)) is bit-exact.
//   * Mapper checkpoint: magic "PKVC", u32 version, the
//     ModelGeometry and MapperConfig, a tensor directory (name, element count,
//     offset) in named_parameters()/named_buffers() order, then the fp64 LE
//     payload — exactly the blob pkv_mapper_create takes, so a trained mapper
//     loads into the B200 path.
// Byte-level semantics follow the reference's binio.hpp (LE u32/u64/f32/f64,
// truncation reported with what was being read); corrupt files map onto its
// IoError taxonomy (common.hpp:33-52): BadMagicError, VersionMismatchError,
// TruncatedFileError, PayloadLengthError. Host code only (no device).
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "mapper.h"

namespace pkv {
namespace {

constexpr uint32_t kTraceVersion = 1, kCkptVersion = 1;

void put_u32(std::ostream& os, uint32_t v) {
    const unsigned char b[4] = {(unsigned char)v, (unsigned char)(v >> 8), (unsigned char)(v >> 16),
                                (unsigned char)(v >> 24)};
    os.write(reinterpret_cast<const char*>(b), 4);
}
void put_u64(std::ostream& os, uint64_t v) {
    put_u32(os, (uint32_t)v);
    put_u32(os, (uint32_t)(v >> 32));
}
// the payload is written element-wise LE (host order on x86/ARM LE; portable)
template <typename T>
void put_array(std::ostream& os, const T* p, size_t n) {
    for (size_t i = 0; i < n; ++i) {
        unsigned char b[sizeof(T)];
        std::memcpy(b, p + i, sizeof(T));
        os.write(reinterpret_cast<const char*>(b), sizeof(T));
    }
}

struct Reader {
    std::ifstream is;
    std::string path;
    uint64_t size = 0, pos = 0;
    explicit Reader(const char* p) : is(p, std::ios::binary), path(p) {
        PKV_REQUIRE(is.good(), PKV_EIO, "cannot open '", p, "'");
        is.seekg(0, std::ios::end);
        size = (uint64_t)is.tellg();
        is.seekg(0);
    }
    void need(uint64_t n, const char* what) {
        PKV_REQUIRE(pos + n <= size, PKV_EIO_TRUNCATED, "file truncated while reading ", what, ": need ", n,
                    " bytes at offset ", pos, ", file has ", size);
    }
    void bytes(void* dst, uint64_t n, const char* what) {
        need(n, what);
        is.read(static_cast<char*>(dst), (std::streamsize)n);
        pos += n;
    }
    uint32_t u32(const char* what) {
        unsigned char b[4];
        bytes(b, 4, what);
        return (uint32_t)b[0] | (uint32_t)b[1] << 8 | (uint32_t)b[2] << 16 | (uint32_t)b[3] << 24;
    }
    uint64_t u64(const char* what) {
        const uint64_t lo = u32(what);
        return lo | (uint64_t)u32(what) << 32;
    }
    void magic(const char* m) {
        char b[4];
        bytes(b, 4, "magic");
        PKV_REQUIRE(std::memcmp(b, m, 4) == 0, PKV_EIO_MAGIC, "bad magic in '", path, "': expected ", m);
    }
};

struct TraceHeader {
    int64_t Ls = 0, Hs = 0, Ll = 0, Hl = 0, N = 0, B = 0, samples = 0;
    std::string meta;
    int64_t x_elems() const { return B * Ls * Hs * N; }
    int64_t y_elems() const { return B * Ll * Hl * N; }
};

TraceHeader read_trace_header(Reader& r) {
    r.magic("PKVT");
    const uint32_t v = r.u32("format version");
    PKV_REQUIRE(v == kTraceVersion, PKV_EIO_VERSION, "trace format version ", v, " (reader supports ", kTraceVersion,
                ")");
    const uint64_t hl = r.u64("header length");
    r.need(hl, "header");  // before sizing anything from the file's own fields
    std::string text(hl, '\0');
    r.bytes(text.data(), hl, "header");
    TraceHeader h;
    std::map<std::string, std::string> kv;
    std::istringstream ss(text);
    std::string line;
    while (std::getline(ss, line)) {
        const auto eq = line.find('=');
        if (eq != std::string::npos) kv[line.substr(0, eq)] = line.substr(eq + 1);
    }
    auto geti = [&](const char* k) {
        auto it = kv.find(k);
        PKV_REQUIRE(it != kv.end(), PKV_EIO, "trace header lacks '", k, "'");
        const char* b = it->second.c_str();
        char* e = nullptr;
        errno = 0;
        const long long v = std::strtoll(b, &e, 10);
        PKV_REQUIRE(e != b && *e == '\0' && errno == 0, PKV_EIO, "trace header field '", k, "' is not an integer: '",
                    it->second, "'");
        return (int64_t)v;
    };
    h.Ls = geti("L_s");
    h.Hs = geti("H_s");
    h.Ll = geti("L_l");
    h.Hl = geti("H_l");
    h.N = geti("N");
    h.B = geti("B");
    h.samples = geti("samples");
    PKV_REQUIRE(kv.count("dtype") && kv["dtype"] == "f32", PKV_EIO, "trace dtype must be f32");
    if (kv.count("meta")) h.meta = kv["meta"];
    for (int64_t e : {h.Ls, h.Hs, h.Ll, h.Hl, h.N, h.B})
        PKV_REQUIRE(e > 0 && e < (int64_t(1) << 31), PKV_EIO, "trace header geometry extent ", e, " out of range");
    PKV_REQUIRE(h.samples >= 0, PKV_EIO, "trace header sample count ", h.samples, " is negative");
    const unsigned __int128 per = (unsigned __int128)(h.x_elems() + h.y_elems()) * 4;
    const unsigned __int128 want = per * (unsigned __int128)h.samples;
    PKV_REQUIRE(want == (unsigned __int128)(r.size - r.pos), PKV_EIO_LENGTH, "trace payload is ", r.size - r.pos,
                " bytes, header geometry implies ", (unsigned long long)(want > ~0ull ? ~0ull : (uint64_t)want));
    return h;
}

// guard() for the file readers: anything that is not already a pkv::Error
// (allocation failure on a hostile size field, stream failures) is an
// IoError, never a CUDA error.
template <typename F>
pkv_status guard_io(F&& f) {
    return guard([&] {
        try {
            f();
        } catch (const Error&) {
            throw;
        } catch (const std::exception& e) {
            throw Error{PKV_EIO, cat("I/O error: ", e.what())};
        }
    });
}

}  // namespace
}  // namespace pkv

using namespace pkv;

extern "C" {

pkv_status pkv_trace_write(const char* path, const int64_t* geom6, int64_t samples, const float* x, const float* y,
                           const char* meta) {
    return guard([&] {
        PKV_REQUIRE_VALUE(path && geom6 && (samples == 0 || (x && y)), "null trace argument");
        for (int i = 0; i < 6; ++i) PKV_REQUIRE_VALUE(geom6[i] > 0, "trace geometry extents must be positive");
        PKV_REQUIRE_VALUE(samples >= 0, "negative sample count");
        std::ostringstream hdr;
        hdr << "L_s=" << geom6[0] << "\nH_s=" << geom6[1] << "\nL_l=" << geom6[2] << "\nH_l=" << geom6[3]
            << "\nN=" << geom6[4] << "\nB=" << geom6[5] << "\ndtype=f32\nsamples=" << samples << "\n";
        if (meta && *meta) {
            std::string m(meta);
            for (char& c : m)
                if (c == '\n') c = ' ';
            hdr << "meta=" << m << "\n";
        }
        const std::string h = hdr.str();
        std::ofstream os(path, std::ios::binary | std::ios::trunc);
        PKV_REQUIRE(os.good(), PKV_EIO, "cannot open '", path, "' for writing");
        os.write("PKVT", 4);
        put_u32(os, kTraceVersion);
        put_u64(os, h.size());
        os.write(h.data(), (std::streamsize)h.size());
        const int64_t nx = geom6[5] * geom6[0] * geom6[1] * geom6[4], ny = geom6[5] * geom6[2] * geom6[3] * geom6[4];
        for (int64_t s = 0; s < samples; ++s) {
            put_array(os, x + s * nx, (size_t)nx);
            put_array(os, y + s * ny, (size_t)ny);
        }
        PKV_REQUIRE(os.good(), PKV_EIO, "write to '", path, "' failed");
    });
}

pkv_status pkv_trace_read_header(const char* path, int64_t* geom6_out, int64_t* samples_out) {
    return guard_io([&] {
        Reader r(path);
        const TraceHeader h = read_trace_header(r);
        const int64_t g[6] = {h.Ls, h.Hs, h.Ll, h.Hl, h.N, h.B};
        for (int i = 0; i < 6; ++i) geom6_out[i] = g[i];
        *samples_out = h.samples;
    });
}

pkv_status pkv_trace_read(const char* path, float* x_out, float* y_out) {
    return guard_io([&] {
        Reader r(path);
        const TraceHeader h = read_trace_header(r);
        for (int64_t s = 0; s < h.samples; ++s) {
            r.bytes(x_out + s * h.x_elems(), (uint64_t)h.x_elems() * 4, "X payload");
            r.bytes(y_out + s * h.y_elems(), (uint64_t)h.y_elems() * 4, "Y payload");
        }
    });
}

pkv_status pkv_checkpoint_write(const char* path, const int64_t* geom5, const int64_t* cfg12, const double* blob,
                                int64_t count) {
    return guard([&] {
        const Geometry g = Geometry::from5(geom5);
        const Config c = Config::from12(cfg12);
        g.validate();
        c.validate();
        const auto layout = param_layout(g, c);
        int64_t total = 0;
        for (const auto& e : layout) total += e.second;
        PKV_REQUIRE_VALUE(total == count, "parameter blob has ", count, " values, layout expects ", total);
        std::ofstream os(path, std::ios::binary | std::ios::trunc);
        PKV_REQUIRE(os.good(), PKV_EIO, "cannot open '", path, "' for writing");
        os.write("PKVC", 4);
        put_u32(os, kCkptVersion);
        for (int i = 0; i < 5; ++i) put_u64(os, (uint64_t)geom5[i]);
        for (int i = 0; i < 12; ++i) put_u64(os, (uint64_t)cfg12[i]);
        put_u64(os, layout.size());
        int64_t off = 0;
        for (const auto& [name, n] : layout) {
            put_u32(os, (uint32_t)name.size());
            os.write(name.data(), (std::streamsize)name.size());
            put_u64(os, (uint64_t)n);
            put_u64(os, (uint64_t)off);
            off += n;
        }
        put_array(os, blob, (size_t)count);
        PKV_REQUIRE(os.good(), PKV_EIO, "write to '", path, "' failed");
    });
}

pkv_status pkv_checkpoint_read(const char* path, int64_t* geom5_out, int64_t* cfg12_out, double* blob_out,
                               int64_t* count_out) {
    return guard_io([&] {
        Reader r(path);
        r.magic("PKVC");
        const uint32_t v = r.u32("format version");
        PKV_REQUIRE(v == kCkptVersion, PKV_EIO_VERSION, "checkpoint format version ", v, " (reader supports ",
                    kCkptVersion, ")");
        int64_t g5[5], c12[12];
        for (auto& x : g5) x = (int64_t)r.u64("geometry");
        for (auto& x : c12) x = (int64_t)r.u64("mapper config");
        const Geometry g = Geometry::from5(g5);
        const Config c = Config::from12(c12);
        g.validate();
        c.validate();
        const auto layout = param_layout(g, c);
        const uint64_t nt = r.u64("tensor count");
        PKV_REQUIRE(nt == layout.size(), PKV_EIO_LENGTH, "checkpoint directory has ", nt,
                    " tensors, the geometry / config imply ", layout.size());
        int64_t total = 0;
        for (const auto& [name, n] : layout) {
            const uint32_t len = r.u32("tensor name length");
            r.need(len, "tensor name");
            std::string nm(len, '\0');
            r.bytes(nm.data(), len, "tensor name");
            const int64_t cnt = (int64_t)r.u64("tensor size"), off = (int64_t)r.u64("tensor offset");
            PKV_REQUIRE(nm == name && cnt == n && off == total, PKV_EIO_LENGTH, "checkpoint tensor '", nm, "' (", cnt,
                        " values at ", off, ") does not match the layout entry '", name, "' (", n, " at ", total,
                        ")");
            total += n;
        }
        PKV_REQUIRE(r.size - r.pos == (uint64_t)total * 8, PKV_EIO_LENGTH, "checkpoint payload is ", r.size - r.pos,
                    " bytes, the directory implies ", total * 8);
        for (int i = 0; i < 5; ++i) geom5_out[i] = g5[i];
        for (int i = 0; i < 12; ++i) cfg12_out[i] = c12[i];
        *count_out = total;
        if (blob_out) r.bytes(blob_out, (uint64_t)total * 8, "payload");
    });
}

}  // extern "C"
