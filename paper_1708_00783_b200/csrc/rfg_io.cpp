// rfg_io.cpp — Netpbm IO of depth / colour frames (proj/src/image_io.cpp),
// host side.  The header grammar and error messages follow the reference:
// a token skips whitespace and '#' comment lines and consumes exactly one
// whitespace byte after itself (image_io.cpp:13-30), so the pixel payload
// starts right after the maxval token.  PGM16 payloads are big-endian
// (image_io.cpp:78-94); rfg_read_pgm16_payload hands them over unconverted so
// the byte swap happens on the GPU inside the depth conversion
// (rfg_view.cu:k_depth_convert, rfg_build_view raw_big_endian = 1).
#include <cctype>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/rfg.h"

namespace rfg {
void set_error(const std::string& msg);
}

namespace {

struct File {
  FILE* f = nullptr;
  explicit File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
  ~File() {
    if (f) std::fclose(f);
  }
};

// pnmToken (image_io.cpp:13-30); false on end of header
bool pnm_token(FILE* f, std::string& tok) {
  tok.clear();
  int c;
  while ((c = std::fgetc(f)) != EOF) {
    if (c == '#') {
      while ((c = std::fgetc(f)) != EOF && c != '\n') {
      }
      continue;
    }
    if (!std::isspace(c)) {
      tok.push_back(static_cast<char>(c));
      break;
    }
  }
  while ((c = std::fgetc(f)) != EOF && !std::isspace(c)) tok.push_back(static_cast<char>(c));
  return !tok.empty();
}

int fail(int code, const std::string& msg) {
  rfg::set_error(msg);
  return code;
}

// header of a P5 / P6 file; returns RFG_OK and leaves f at the payload
int pnm_header(FILE* f, const char* path, const char* magic, int wantMax, const char* kind, int* w, int* h) {
  std::string tok;
  if (!pnm_token(f, tok)) return fail(RFG_EINVAL, "pnm: unexpected end of header");
  if (tok != magic)
    return fail(RFG_EINVAL, std::string("not a binary ") + kind + " (" + magic + "): " + path);
  int v[3];
  for (int k = 0; k < 3; ++k) {
    if (!pnm_token(f, tok)) return fail(RFG_EINVAL, "pnm: unexpected end of header");
    char* end = nullptr;
    const long x = std::strtol(tok.c_str(), &end, 10);  // std::stoi: leading integer prefix
    if (end == tok.c_str()) return fail(RFG_EINVAL, "stoi");
    v[k] = static_cast<int>(x);
  }
  *w = v[0];
  *h = v[1];
  if (v[2] != wantMax)
    return fail(RFG_EINVAL, std::string("unsupported ") + kind + " maxval (want " + std::to_string(wantMax) +
                                "): " + path);
  if (v[0] < 0 || v[1] < 0) return fail(RFG_EINVAL, std::string("invalid ") + kind + " size: " + path);
  return RFG_OK;
}

int read_pgm_bytes(const char* path, void* out, int64_t capacity, int* w, int* h, bool swap) {
  if (!path || !w || !h) return fail(RFG_EINVAL, "null argument");
  File f(path, "rb");
  if (!f.f) return fail(RFG_EINVAL, std::string("cannot open ") + path);
  int rc = pnm_header(f.f, path, "P5", 65535, "PGM", w, h);
  if (rc != RFG_OK) return rc;
  const int64_t n = (int64_t)*w * *h;
  if (!out || n > capacity) return fail(RFG_ERANGE, "pgm: output capacity too small");
  const size_t bytes = (size_t)n * 2;
  if (std::fread(out, 1, bytes, f.f) != bytes) return fail(RFG_EINVAL, std::string("truncated PGM: ") + path);
  if (swap) {
    uint8_t* b = static_cast<uint8_t*>(out);
    uint16_t* o = static_cast<uint16_t*>(out);
    for (int64_t i = 0; i < n; ++i) o[i] = static_cast<uint16_t>((b[2 * i] << 8) | b[2 * i + 1]);
  }
  return RFG_OK;
}

}  // namespace

extern "C" {

int rfg_read_pgm16(const char* path, uint16_t* out, int64_t capacity, int* width, int* height) {
  return read_pgm_bytes(path, out, capacity, width, height, true);
}

int rfg_read_pgm16_payload(const char* path, void* out, int64_t capacity, int* width, int* height) {
  return read_pgm_bytes(path, out, capacity, width, height, false);
}

int rfg_read_ppm(const char* path, uint8_t* out, int64_t capacity, int* width, int* height) {
  if (!path || !width || !height) return fail(RFG_EINVAL, "null argument");
  File f(path, "rb");
  if (!f.f) return fail(RFG_EINVAL, std::string("cannot open ") + path);
  int rc = pnm_header(f.f, path, "P6", 255, "PPM", width, height);
  if (rc != RFG_OK) return rc;
  const int64_t n = (int64_t)*width * *height;
  if (!out || n > capacity) return fail(RFG_ERANGE, "ppm: output capacity too small");
  const size_t bytes = (size_t)n * 3;
  if (std::fread(out, 1, bytes, f.f) != bytes) return fail(RFG_EINVAL, std::string("truncated PPM: ") + path);
  return RFG_OK;
}

int rfg_write_pgm16(const char* path, const uint16_t* img, int width, int height) {
  if (!path || (!img && width * height > 0) || width < 0 || height < 0) return fail(RFG_EINVAL, "null argument");
  File f(path, "wb");
  if (!f.f) return fail(RFG_EINVAL, std::string("cannot write ") + path);
  std::fprintf(f.f, "P5\n%d %d\n65535\n", width, height);
  std::vector<unsigned char> row(static_cast<size_t>(width) * 2);
  for (int y = 0; y < height; ++y) {
    for (int x = 0; x < width; ++x) {
      const uint16_t v = img[(size_t)y * width + x];
      row[2 * x] = static_cast<unsigned char>(v >> 8);
      row[2 * x + 1] = static_cast<unsigned char>(v & 0xFF);
    }
    if (std::fwrite(row.data(), 1, row.size(), f.f) != row.size())
      return fail(RFG_EINVAL, std::string("short write: ") + path);
  }
  return RFG_OK;
}

int rfg_write_ppm(const char* path, const uint8_t* rgb, int width, int height) {
  if (!path || (!rgb && width * height > 0) || width < 0 || height < 0) return fail(RFG_EINVAL, "null argument");
  File f(path, "wb");
  if (!f.f) return fail(RFG_EINVAL, std::string("cannot write ") + path);
  std::fprintf(f.f, "P6\n%d %d\n255\n", width, height);
  const size_t bytes = (size_t)width * height * 3;
  if (std::fwrite(rgb, 1, bytes, f.f) != bytes) return fail(RFG_EINVAL, std::string("short write: ") + path);
  return RFG_OK;
}

}  // extern "C"
