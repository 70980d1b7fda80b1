// io.h — host interface of the cloud IO module (io.cu).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace pcsb {

// A reference ParseError (proj/include/pcs/errors.hpp): 1-based line number and
// reason; the C ABI reports it as PCS_ERR_PARSE + pcs_parse_error.
struct ParseFailure : std::runtime_error {
    int64_t line;
    std::string reason;
    ParseFailure(int64_t l, const std::string& r) : std::runtime_error(r), line(l), reason(r) {}
};

struct PlyHeader {
    struct Element {
        std::string name;
        long count = 0;
        std::vector<std::string> props;
        bool has_list = false;
    };
    std::vector<Element> elements;
    int64_t header_lines = 0;
    uint64_t body = 0;  // byte offset of the first body line
};

PlyHeader ply_header(const char* text, uint64_t len);

// Text of write_cloud_stream (format: PCS_FMT_*); returns the byte count; writes
// only when out has room (cap >= count).
uint64_t format_cloud(const double* xyz, uint64_t n, int format, char* out, uint64_t cap);
// Same, one pass, into a malloc'd buffer (*out, freed by the caller with free()).
uint64_t format_cloud_alloc(const double* xyz, uint64_t n, int format, char** out);
// read_cloud_stream: xyz of the points; throws ParseFailure.
// Caller-side destination of parse_cloud: when the parsed points fit `cap`, they
// are copied from the device straight into `ext` (used = true, n = points) and
// the returned vector stays empty — no intermediate host copy.
struct ParseDst {
    double* ext = nullptr;
    uint64_t cap = 0;
    bool used = false;
    uint64_t n = 0;
};
std::vector<double> parse_cloud(const char* text, uint64_t len, int format, ParseDst* dst = nullptr);
// read_mesh_stream: 9 doubles per triangle (fan-triangulated faces); throws ParseFailure.
std::vector<double> parse_mesh(const char* text, uint64_t len);

}  // namespace pcsb
