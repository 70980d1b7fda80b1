// io.cu — point-cloud text IO on the device (the data
// format either side of the LOP path).
//
// Replaces the reference's
//   write_cloud_stream   proj/src/io.cpp:277-290  (XYZ / ASCII PLY, coordinates
//                        printed by format_double = std::to_chars shortest
//                        round-trip, :240-245)
//   read_cloud_stream    proj/src/io.cpp:260-264  (read_xyz :143-165,
//                        read_ply :171-236, parse_double = std::from_chars :36-48)
// byte-for-byte (writer) and bit-for-bit with identical ParseError lines and
// reasons (reader).
//
// Writer: one thread per point formats "x y z\n" twice — once for its length,
// once into place after an exclusive scan of the lengths — with csrc/dconv.h.
// Reader: line starts are found by a flag + stream compaction over the bytes;
// one thread per line classifies it (blank / comment / data, with the
// reference's isspace set) and parses its tokens with dconv::parse; an exclusive
// scan of the data flags places each point.  A line the device cannot settle (a
// malformed line, a number beyond the exact fast path) is re-read on the host
// with the reference's semantics, so errors carry the reference's line number
// and reason.  PLY headers, meshes and every PLY anomaly (short files, header
// errors) take the host path, which implements the complete format.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>
#include <cctype>
#include <charconv>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "dconv.h"
#include "host_io.h"
#include "io.h"
#include "plan.cuh"

namespace pcsb {

// ---- host side: the reference's text semantics ---------------------------------
namespace {

inline bool is_ws(char c) {  // std::isspace in the "C" locale
    return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

std::vector<std::string> tokens_of(const char* b, const char* e) {
    std::vector<std::string> t;
    while (b < e) {
        while (b < e && is_ws(*b)) ++b;
        const char* s = b;
        while (b < e && !is_ws(*b)) ++b;
        if (b > s) t.emplace_back(s, b);
    }
    return t;
}

bool blank(const char* b, const char* e) {
    for (; b < e; ++b)
        if (!is_ws(*b)) return false;
    return true;
}

[[noreturn]] void fail(int64_t line, const std::string& reason) { throw ParseFailure(line, reason); }

double host_double(const std::string& tok, int64_t line) {
    double v = 0.0;
    const char* b = tok.data();
    const char* e = b + tok.size();
    const auto r = std::from_chars(b, e, v);
    if (r.ec == std::errc::result_out_of_range) fail(line, "number out of range: '" + tok + "'");
    if (r.ec != std::errc() || r.ptr != e) fail(line, "not a number: '" + tok + "'");
    if (!std::isfinite(v)) fail(line, "non-finite coordinate: '" + tok + "'");
    return v;
}

long host_long(const std::string& tok, int64_t line) {
    long v = 0;
    const char* b = tok.data();
    const char* e = b + tok.size();
    const auto r = std::from_chars(b, e, v);
    if (r.ec != std::errc() || r.ptr != e || v < 0)
        fail(line, "not a non-negative integer: '" + tok + "'");
    return v;
}

// Physical lines (getline semantics: split on '\n', a last line without '\n'
// counts, nothing after a final '\n').
struct Lines {
    const char* t;
    uint64_t len, pos = 0;
    int64_t no = 0;
    bool next(const char*& b, const char*& e) {
        if (pos >= len) return false;
        b = t + pos;
        const void* nl = std::memchr(b, '\n', len - pos);
        e = nl ? (const char*)nl : t + len;
        pos = (uint64_t)(e - t) + (nl ? 1 : 0);
        ++no;
        if (e > b && e[-1] == '\r') --e;  // rtrim_cr
        return true;
    }
};

// XYZ data line (proj/src/io.cpp:150-162)
void xyz_line(const char* b, const char* e, int64_t line, double* out) {
    const auto tk = tokens_of(b, e);
    if (tk.size() != 3) fail(line, "expected 3 coordinates, got " + std::to_string(tk.size()));
    out[0] = host_double(tk[0], line);
    out[1] = host_double(tk[1], line);
    out[2] = host_double(tk[2], line);
}

}  // namespace

PlyHeader ply_header(const char* t, uint64_t len) {
    PlyHeader h;
    Lines L{t, len};
    const char *b, *e;
    if (!L.next(b, e)) throw ParseFailure(1, "empty file, expected 'ply'");
    if (std::string(b, e) != "ply") throw ParseFailure(1, "missing 'ply' magic line");
    bool format_seen = false, ended = false;
    while (L.next(b, e)) {
        const auto tk = tokens_of(b, e);
        const int64_t no = L.no;
        if (tk.empty()) fail(no, "blank line inside header");
        if (tk[0] == "comment" || tk[0] == "obj_info") continue;
        if (tk[0] == "format") {
            if (tk.size() != 3 || tk[1] != "ascii") fail(no, "only 'format ascii 1.0' is supported");
            format_seen = true;
        } else if (tk[0] == "element") {
            if (tk.size() != 3) fail(no, "malformed element line");
            PlyHeader::Element el;
            el.name = tk[1];
            el.count = host_long(tk[2], no);
            h.elements.push_back(el);
        } else if (tk[0] == "property") {
            if (h.elements.empty()) fail(no, "property before any element");
            if (tk.size() >= 2 && tk[1] == "list") {
                if (tk.size() != 5) fail(no, "malformed list property");
                h.elements.back().has_list = true;
            } else {
                if (tk.size() != 3) fail(no, "malformed property line");
                h.elements.back().props.push_back(tk[2]);
            }
        } else if (tk[0] == "end_header") {
            ended = true;
            break;
        } else {
            fail(no, "unknown header keyword '" + tk[0] + "'");
        }
    }
    if (!ended) fail(L.no, "header not terminated by end_header");
    if (!format_seen) fail(L.no, "header missing format line");
    h.header_lines = L.no;
    h.body = L.pos;
    return h;
}

// The complete PLY body on the host (proj/src/io.cpp:171-236): vertices and,
// when wanted, faces.
void ply_host(const char* t, uint64_t len, bool want_faces, std::vector<double>& xyz,
              std::vector<std::vector<long>>* faces) {
    const PlyHeader h = ply_header(t, len);
    Lines L{t, len};
    L.pos = h.body;
    L.no = h.header_lines;
    const char *b, *e;
    auto data_line = [&](const char* what) {
        while (L.next(b, e))
            if (!blank(b, e)) return;
        fail(L.no, std::string("unexpected end of file reading ") + what);
    };
    bool vertex_seen = false;
    for (const auto& el : h.elements) {
        if (el.name == "vertex") {
            vertex_seen = true;
            if (el.has_list) fail(L.no, "list property in vertex element unsupported");
            auto find = [&](const char* p) {
                const auto it = std::find(el.props.begin(), el.props.end(), p);
                if (it == el.props.end())
                    fail(L.no, std::string("vertex element lacks property ") + p);
                return (size_t)(it - el.props.begin());
            };
            const size_t ix = find("x"), iy = find("y"), iz = find("z");
            for (long i = 0; i < el.count; ++i) {
                data_line("vertex");
                const auto tk = tokens_of(b, e);
                if (tk.size() != el.props.size())
                    fail(L.no, "expected " + std::to_string(el.props.size()) + " vertex values, got " +
                                   std::to_string(tk.size()));
                xyz.push_back(host_double(tk[ix], L.no));
                xyz.push_back(host_double(tk[iy], L.no));
                xyz.push_back(host_double(tk[iz], L.no));
            }
        } else if (el.name == "face" && want_faces) {
            if (!el.has_list) fail(L.no, "face element lacks a list property");
            for (long i = 0; i < el.count; ++i) {
                data_line("face");
                const auto tk = tokens_of(b, e);
                if (tk.empty()) fail(L.no, "empty face line");
                const long arity = host_long(tk[0], L.no);
                if (arity < 3) fail(L.no, "face with fewer than 3 vertices");
                if ((long)tk.size() != arity + 1) fail(L.no, "face vertex count mismatch");
                std::vector<long> f((size_t)arity);
                for (long k = 0; k < arity; ++k) f[(size_t)k] = host_long(tk[(size_t)k + 1], L.no);
                faces->push_back(std::move(f));
            }
        } else {
            for (long i = 0; i < el.count; ++i) data_line(el.name.c_str());
        }
    }
    if (!vertex_seen) fail(L.no, "no vertex element in file");
}

// ---- device kernels -------------------------------------------------------------
namespace {

constexpr int IO_THREADS = 256;

__device__ __forceinline__ bool d_ws(char c) {
    return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

__device__ __forceinline__ int point_text(const double* p, char* o) {
    int n = dconv::format(p[0], o);
    o[n++] = ' ';
    n += dconv::format(p[1], o + n);
    o[n++] = ' ';
    n += dconv::format(p[2], o + n);
    o[n++] = '\n';
    return n;
}

__global__ void fmt_len_kernel(const double* __restrict__ xyz, uint64_t n, uint64_t* __restrict__ len) {
    const uint64_t i = (uint64_t)blockIdx.x * IO_THREADS + threadIdx.x;
    if (i >= n) return;
    char buf[96];
    len[i] = (uint64_t)point_text(xyz + 3 * i, buf);
}

__global__ void fmt_write_kernel(const double* __restrict__ xyz, uint64_t n,
                                 const uint64_t* __restrict__ off, char* __restrict__ out) {
    const uint64_t i = (uint64_t)blockIdx.x * IO_THREADS + threadIdx.x;
    if (i >= n) return;
    char buf[96];
    const int m = point_text(xyz + 3 * i, buf);
    char* o = out + off[i];
    for (int k = 0; k < m; ++k) o[k] = buf[k];
}

__global__ void line_flag_kernel(const char* __restrict__ t, uint64_t len, uint8_t* __restrict__ f) {
    const uint64_t i = (uint64_t)blockIdx.x * IO_THREADS + threadIdx.x;
    if (i < len) f[i] = (i == 0 || t[i - 1] == '\n') ? 1 : 0;
}

struct LineSpan {
    uint64_t b, e;
};

__device__ __forceinline__ LineSpan line_span(const char* t, uint64_t len, const uint64_t* starts,
                                              uint64_t nl, uint64_t k) {
    const uint64_t b = starts[k];
    uint64_t e = k + 1 < nl ? starts[k + 1] - 1 : len;  // exclude '\n'
    if (k + 1 >= nl && e > b && t[e - 1] == '\n') --e;
    return {b, e};
}

struct Widen {
    __host__ __device__ __forceinline__ uint64_t operator()(uint8_t v) const { return v; }
};

struct IsHost {
    __host__ __device__ __forceinline__ uint8_t operator()(uint8_t s) const { return s == 2 ? 1 : 0; }
};

// cls: 0 = not a data line; 1 = data line.  XYZ: blank or '#' comment lines are
// skipped (io.cpp:148-153); PLY body: only blank lines (next_data_line).
__global__ void line_class_kernel(const char* __restrict__ t, uint64_t len,
                                  const uint64_t* __restrict__ starts, uint64_t nl, int ply,
                                  uint64_t* __restrict__ cls) {
    const uint64_t k = (uint64_t)blockIdx.x * IO_THREADS + threadIdx.x;
    if (k >= nl) return;
    const LineSpan s = line_span(t, len, starts, nl, k);
    uint64_t p = s.b;
    while (p < s.e && d_ws(t[p])) ++p;
    uint64_t c = p < s.e ? 1u : 0u;
    if (c && !ply) {
        uint64_t q = s.b;
        while (q < s.e && (t[q] == ' ' || t[q] == '\t')) ++q;
        if (q < s.e && t[q] == '#') c = 0;
    }
    cls[k] = c;
}

// Parses the data lines: XYZ (ntok = 3, slots 0,1,2) or a PLY vertex range (ntok =
// the element's property count, slots ix, iy, iz; data ordinals [o0, o0 + cnt)).
// st: 0 = not a point line, 1 = parsed, 2 = leave to the host.
__global__ void line_parse_kernel(const char* __restrict__ t, uint64_t len,
                                  const uint64_t* __restrict__ starts, uint64_t nl,
                                  const uint64_t* __restrict__ cls, const uint64_t* __restrict__ ord,
                                  int ntok, int ix, int iy, int iz, uint64_t o0, uint64_t cnt,
                                  double* __restrict__ xyz, uint8_t* __restrict__ st) {
    const uint64_t k = (uint64_t)blockIdx.x * IO_THREADS + threadIdx.x;
    if (k >= nl) return;
    uint8_t s = 0;
    if (cls[k]) {
        const uint64_t o = ord[k];
        if (o >= o0 && o - o0 < cnt) {
            const uint64_t idx = o - o0;
            const LineSpan sp = line_span(t, len, starts, nl, k);
            double v[3] = {0.0, 0.0, 0.0};
            int ntk = 0;
            bool ok = true;
            uint64_t p = sp.b;
            while (p < sp.e) {
                while (p < sp.e && d_ws(t[p])) ++p;
                if (p >= sp.e) break;
                const uint64_t b = p;
                while (p < sp.e && !d_ws(t[p])) ++p;
                const int slot = ntk == ix ? 0 : (ntk == iy ? 1 : (ntk == iz ? 2 : -1));
                if (slot >= 0 && ntk < ntok) {
                    double x;
                    if (dconv::parse(t + b, t + p, &x)) v[slot] = x;
                    else ok = false;
                }
                ++ntk;
            }
            if (ntk != ntok) ok = false;
            if (ok) {
                xyz[3 * idx] = v[0];
                xyz[3 * idx + 1] = v[1];
                xyz[3 * idx + 2] = v[2];
            }
            s = ok ? 1 : 2;
        }
    }
    st[k] = s;
}

struct DevMem {  // stream-ordered temporaries of one call, from the library's pool
    cudaStream_t s;
    int dev = 0;
    std::vector<void*> p;
    explicit DevMem(cudaStream_t s_) : s(s_) { PCSB_CUDA(cudaGetDevice(&dev)); }
    ~DevMem() {
        for (void* x : p) pool_free(x, s);
    }
    template <typename X>
    X* get(size_t count) {
        void* x = pool_alloc(dev, std::max<size_t>(count * sizeof(X), 16), s);
        p.push_back(x);
        return (X*)x;
    }
};

struct IoStream {
    cudaStream_t s = nullptr;
    IoStream() { PCSB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
    ~IoStream() {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
    }
};

unsigned grid_of(uint64_t n) { return (unsigned)((n + IO_THREADS - 1) / IO_THREADS); }

template <typename T>
void exclusive_scan(const T* in, T* out, uint64_t n, DevMem& mem, cudaStream_t s) {
    size_t bytes = 0;
    PCSB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, (int64_t)n, s));
    void* tmp = mem.get<uint8_t>(bytes);
    PCSB_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, (int64_t)n, s));
}

std::string ply_header_text(uint64_t n) {
    return "ply\nformat ascii 1.0\nelement vertex " + std::to_string(n) +
           "\nproperty double x\nproperty double y\nproperty double z\nend_header\n";
}

}  // namespace

// ---- writer ---------------------------------------------------------------------
uint64_t format_cloud(const double* xyz, uint64_t n, int format, char* out, uint64_t cap) {
    const std::string head = format == PCS_FMT_PLY_ASCII ? ply_header_text(n) : std::string();
    if (n == 0) {
        if (out && cap >= head.size()) std::memcpy(out, head.data(), head.size());
        return head.size();
    }
    IoStream st;
    DevMem mem(st.s);
    double* dxyz = mem.get<double>(n * 3);
    uint64_t* len = mem.get<uint64_t>(n + 1);
    uint64_t* off = mem.get<uint64_t>(n + 1);
    h2d_staged(dxyz, xyz, n * 3 * sizeof(double), st.s);
    PCSB_CUDA(cudaMemsetAsync(len + n, 0, sizeof(uint64_t), st.s));
    fmt_len_kernel<<<grid_of(n), IO_THREADS, 0, st.s>>>(dxyz, n, len);
    PCSB_CUDA(cudaGetLastError());
    exclusive_scan(len, off, n + 1, mem, st.s);
    uint64_t body = 0;
    PCSB_CUDA(cudaMemcpyAsync(&body, off + n, sizeof(uint64_t), cudaMemcpyDeviceToHost, st.s));
    PCSB_CUDA(cudaStreamSynchronize(st.s));
    const uint64_t total = head.size() + body;
    if (!out || cap < total) return total;
    char* dout = mem.get<char>(body);
    fmt_write_kernel<<<grid_of(n), IO_THREADS, 0, st.s>>>(dxyz, n, off, dout);
    PCSB_CUDA(cudaGetLastError());
    std::memcpy(out, head.data(), head.size());
    d2h_staged(out + head.size(), dout, body, st.s);
    return total;
}

uint64_t format_cloud_alloc(const double* xyz, uint64_t n, int format, char** out) {
    const std::string head = format == PCS_FMT_PLY_ASCII ? ply_header_text(n) : std::string();
    if (n == 0) {
        *out = (char*)std::malloc(std::max<size_t>(head.size(), 1));
        if (!*out) throw std::bad_alloc();
        std::memcpy(*out, head.data(), head.size());
        return head.size();
    }
    IoStream st;
    DevMem mem(st.s);
    double* dxyz = mem.get<double>(n * 3);
    uint64_t* len = mem.get<uint64_t>(n + 1);
    uint64_t* off = mem.get<uint64_t>(n + 1);
    h2d_staged(dxyz, xyz, n * 3 * sizeof(double), st.s);
    PCSB_CUDA(cudaMemsetAsync(len + n, 0, sizeof(uint64_t), st.s));
    fmt_len_kernel<<<grid_of(n), IO_THREADS, 0, st.s>>>(dxyz, n, len);
    PCSB_CUDA(cudaGetLastError());
    exclusive_scan(len, off, n + 1, mem, st.s);
    uint64_t body = 0;
    PCSB_CUDA(cudaMemcpyAsync(&body, off + n, sizeof(uint64_t), cudaMemcpyDeviceToHost, st.s));
    PCSB_CUDA(cudaStreamSynchronize(st.s));
    char* dout = mem.get<char>(body);
    fmt_write_kernel<<<grid_of(n), IO_THREADS, 0, st.s>>>(dxyz, n, off, dout);
    PCSB_CUDA(cudaGetLastError());
    const uint64_t total = head.size() + body;
    char* h = (char*)std::malloc(total);
    if (!h) throw std::bad_alloc();
    std::memcpy(h, head.data(), head.size());
    d2h_staged(h + head.size(), dout, body, st.s);
    *out = h;
    return total;
}

// ---- reader ---------------------------------------------------------------------
namespace {

// A data line the device left to the host: its physical index, data ordinal
// and byte span (without '\n').
struct HostLine {
    uint64_t k, ord, b, e;
};

__global__ void host_line_kernel(const char* __restrict__ t, uint64_t len,
                                 const uint64_t* __restrict__ starts, uint64_t nl,
                                 const uint64_t* __restrict__ ord, const uint64_t* __restrict__ sel,
                                 const uint64_t* __restrict__ nsel, HostLine* __restrict__ out) {
    const uint64_t i = (uint64_t)blockIdx.x * IO_THREADS + threadIdx.x;
    if (i >= *nsel) return;
    const uint64_t k = sel[i];
    const LineSpan sp = line_span(t, len, starts, nl, k);
    out[i] = {k, ord[k], sp.b, sp.e};
}

// Device pass over [t, t + len): line starts, classes, data ordinals and the
// parse of data ordinals [o0, o0 + cnt) (cnt = ~0: all data lines) into xyz;
// only the lines left to the host come back as HostLine records.
struct DevParse {
    uint64_t nlines = 0, ndata = 0;
    std::vector<HostLine> host;
    double* out = nullptr;  // where the points landed (the caller's buffer or xyz)
};

DevParse device_parse(const char* t, uint64_t len, bool ply, int ntok, int ix, int iy, int iz,
                      uint64_t o0, uint64_t cnt, std::vector<double>& xyz, ParseDst* pdst) {
    DevParse r;
    xyz.clear();
    if (pdst) pdst->used = false;
    if (len == 0) return r;
    IoStream st;
    DevMem mem(st.s);
    char* dt = mem.get<char>(len);
    h2d_staged(dt, t, len, st.s);
    uint8_t* flag = mem.get<uint8_t>(len);
    line_flag_kernel<<<grid_of(len), IO_THREADS, 0, st.s>>>(dt, len, flag);
    PCSB_CUDA(cudaGetLastError());
    uint64_t* nsel = mem.get<uint64_t>(2);
    // count the lines first, so the start table is sized by lines, not bytes
    {
        thrust::transform_iterator<Widen, const uint8_t*> wf(flag, Widen());
        size_t bytes = 0;
        PCSB_CUDA(cub::DeviceReduce::Sum(nullptr, bytes, wf, nsel, (int64_t)len, st.s));
        void* tmp = mem.get<uint8_t>(bytes);
        PCSB_CUDA(cub::DeviceReduce::Sum(tmp, bytes, wf, nsel, (int64_t)len, st.s));
    }
    uint64_t nl_count = 0;
    PCSB_CUDA(cudaMemcpyAsync(&nl_count, nsel, sizeof(uint64_t), cudaMemcpyDeviceToHost, st.s));
    PCSB_CUDA(cudaStreamSynchronize(st.s));
    uint64_t* starts = mem.get<uint64_t>(nl_count + 1);
    auto select = [&](const uint8_t* f, uint64_t n, uint64_t* outsel, uint64_t* count) {
        thrust::counting_iterator<uint64_t> it(0);
        size_t bytes = 0;
        PCSB_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, f, outsel, count, (int64_t)n, st.s));
        void* tmp = mem.get<uint8_t>(bytes);
        PCSB_CUDA(cub::DeviceSelect::Flagged(tmp, bytes, it, f, outsel, count, (int64_t)n, st.s));
    };
    select(flag, len, starts, nsel);
    PCSB_CUDA(cudaMemcpyAsync(&r.nlines, nsel, sizeof(uint64_t), cudaMemcpyDeviceToHost, st.s));
    PCSB_CUDA(cudaStreamSynchronize(st.s));
    const uint64_t nl = r.nlines;
    uint64_t* cls = mem.get<uint64_t>(nl + 1);
    uint64_t* ord = mem.get<uint64_t>(nl + 1);
    PCSB_CUDA(cudaMemsetAsync(cls + nl, 0, sizeof(uint64_t), st.s));
    line_class_kernel<<<grid_of(nl), IO_THREADS, 0, st.s>>>(dt, len, starts, nl, ply ? 1 : 0, cls);
    PCSB_CUDA(cudaGetLastError());
    exclusive_scan(cls, ord, nl + 1, mem, st.s);
    PCSB_CUDA(cudaMemcpyAsync(&r.ndata, ord + nl, sizeof(uint64_t), cudaMemcpyDeviceToHost, st.s));
    PCSB_CUDA(cudaStreamSynchronize(st.s));
    const uint64_t avail = r.ndata > o0 ? r.ndata - o0 : 0;
    const uint64_t npts = std::min(cnt, avail);
    double* dxyz = mem.get<double>(npts * 3);
    uint8_t* dst = mem.get<uint8_t>(nl);
    line_parse_kernel<<<grid_of(nl), IO_THREADS, 0, st.s>>>(dt, len, starts, nl, cls, ord, ntok, ix, iy,
                                                          iz, o0, npts, dxyz, dst);
    PCSB_CUDA(cudaGetLastError());
    // the lines left to the host: st == 2 (flag bytes reused)
    uint64_t* hsel = mem.get<uint64_t>(nl);
    HostLine* hl = mem.get<HostLine>(nl);
    {
        uint8_t* f2 = flag;  // nl <= len
        thrust::transform_iterator<IsHost, const uint8_t*> fi(dst, IsHost());
        size_t bytes = 0;
        thrust::counting_iterator<uint64_t> it(0);
        (void)f2;
        PCSB_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, fi, hsel, nsel + 1, (int64_t)nl, st.s));
        void* tmp = mem.get<uint8_t>(bytes);
        PCSB_CUDA(cub::DeviceSelect::Flagged(tmp, bytes, it, fi, hsel, nsel + 1, (int64_t)nl, st.s));
    }
    host_line_kernel<<<grid_of(nl), IO_THREADS, 0, st.s>>>(dt, len, starts, nl, ord, hsel, nsel + 1, hl);
    PCSB_CUDA(cudaGetLastError());
    uint64_t nhost = 0;
    PCSB_CUDA(cudaMemcpyAsync(&nhost, nsel + 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, st.s));
    if (pdst && pdst->ext && npts <= pdst->cap) {
        pdst->used = true;
        pdst->n = npts;
        r.out = pdst->ext;
    } else {
        xyz.resize(npts * 3);
        r.out = xyz.data();
    }
    PCSB_CUDA(cudaStreamSynchronize(st.s));
    if (npts) d2h_staged(r.out, dxyz, npts * 3 * sizeof(double), st.s);
    r.host.resize(nhost);
    if (nhost)
        PCSB_CUDA(cudaMemcpyAsync(r.host.data(), hl, nhost * sizeof(HostLine), cudaMemcpyDeviceToHost, st.s));
    PCSB_CUDA(cudaStreamSynchronize(st.s));
    PCSB_CUDA(cudaGetLastError());
    return r;
}

}  // namespace

std::vector<double> parse_cloud(const char* t, uint64_t len, int format, ParseDst* dst) {
    std::vector<double> xyz;
    if (format == PCS_FMT_XYZ) {
        const DevParse dp = device_parse(t, len, false, 3, 0, 1, 2, 0, ~0ull, xyz, dst);
        // lines the device left to the host, in file order (the first error wins)
        for (const HostLine& h : dp.host) {
            const char* b = t + h.b;
            const char* e = t + h.e;
            if (e > b && e[-1] == '\r') --e;
            xyz_line(b, e, (int64_t)h.k + 1, dp.out + 3 * h.ord);
        }
        return xyz;
    }
    // PLY: header on the host; the vertex element's lines on the device when the
    // file is well formed, else the complete host parser (exact errors)
    const PlyHeader h = ply_header(t, len);
    uint64_t off = 0, total = 0;
    const PlyHeader::Element* vx = nullptr;
    for (const auto& el : h.elements) {
        if (!vx && el.name == "vertex") {
            vx = &el;
            off = total;
        }
        total += (uint64_t)el.count;
    }
    bool simple = vx && !vx->has_list;
    int ix = -1, iy = -1, iz = -1;
    if (simple) {
        auto find = [&](const char* p) {
            const auto it = std::find(vx->props.begin(), vx->props.end(), p);
            return it == vx->props.end() ? -1 : (int)(it - vx->props.begin());
        };
        ix = find("x");
        iy = find("y");
        iz = find("z");
        simple = ix >= 0 && iy >= 0 && iz >= 0;
    }
    if (simple) {
        const uint64_t cnt = (uint64_t)vx->count;
        const DevParse dp = device_parse(t + h.body, len - h.body, true, (int)vx->props.size(), ix, iy,
                                         iz, off, cnt, xyz, dst);
        if (dp.ndata >= total && dp.host.empty()) return xyz;
    }
    xyz.clear();
    if (dst) dst->used = false;
    ply_host(t, len, false, xyz, nullptr);
    return xyz;
}

std::vector<double> parse_mesh(const char* t, uint64_t len) {
    std::vector<double> xyz;
    std::vector<std::vector<long>> faces;
    ply_host(t, len, true, xyz, &faces);
    if (faces.empty()) throw ParseFailure(0, "no face element (or zero faces) in mesh file");
    const long nv = (long)(xyz.size() / 3);
    std::vector<double> tri;
    for (const auto& f : faces) {
        for (long i : f)
            if (i >= nv)
                throw ParseFailure(0, "face references vertex " + std::to_string(i) +
                                          " beyond vertex count");
        for (size_t k = 1; k + 1 < f.size(); ++k)
            for (long v : {f[0], f[k], f[k + 1]})
                for (int a = 0; a < 3; ++a) tri.push_back(xyz[(size_t)v * 3 + a]);
    }
    return tri;
}

}  // namespace pcsb
