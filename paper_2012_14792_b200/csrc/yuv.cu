// Raw planar 4:2:0 YUV ingest (texture.cpp:9-81: yuv_frame_count,
// load_yuv_frame), B200 side: only the luma planes are read (pread at each
// frame's offset, chroma skipped), into pinned staging, and they stay in
// their file format -- uint8 for 8-bit, uint16 little-endian for 10-bit -- so
// K1 reads them natively with no widening pass.  load_yuv_frame's widened
// uint16 plane is still offered for the drop-in LumaPlane (sc_yuv_load_luma).
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cerrno>
#include <cstring>

#include "common.cuh"

namespace scb {

int yuv_bytes_per_sample(int bit_depth) {
  if (bit_depth == 8) return 1;
  if (bit_depth == 10) return 2;
  fail(SC_ERR_FORMAT, "bit depth must be 8 or 10, got " + std::to_string(bit_depth));
}

// frame_bytes (texture.cpp:16-21): luma + two (w+1)/2 x (h+1)/2 chroma planes.
uint64_t yuv_frame_bytes(int w, int h, int bit_depth) {
  const uint64_t luma = (uint64_t)w * h;
  const uint64_t chroma = 2ull * ((uint64_t)((w + 1) / 2) * ((h + 1) / 2));
  return (luma + chroma) * (uint64_t)yuv_bytes_per_sample(bit_depth);
}

// yuv_frame_count (texture.cpp:25-40).
int yuv_frame_count(const char* path, int w, int h, int bit_depth) {
  if (w < 1 || h < 1) fail(SC_ERR_FORMAT, "frame dimensions must be positive");
  struct stat st;
  if (::stat(path, &st) != 0)
    fail(SC_ERR_IO, std::string("cannot stat ") + path + ": " + std::strerror(errno));
  const uint64_t size = (uint64_t)st.st_size, fb = yuv_frame_bytes(w, h, bit_depth);
  if (size % fb != 0)
    fail(SC_ERR_FORMAT, std::string(path) + ": file size " + std::to_string(size) +
                            " is not a multiple of the frame size " + std::to_string(fb));
  return (int)(size / fb);
}

// Raw luma planes of frames [first, first + n) into dst (n * w * h * bps bytes).
void yuv_read_luma(const char* path, int w, int h, int bit_depth, int first, int n, void* dst) {
  const int frames = yuv_frame_count(path, w, h, bit_depth);
  if (n < 1) fail(SC_ERR_USAGE, "n_frames must be >= 1");
  if (first < 0 || first + n > frames)
    fail(SC_ERR_RANGE, std::string(path) + ": frame " +
                           std::to_string(first < 0 ? first : first + n - 1) +
                           " out of range, file holds " + std::to_string(frames));
  const int fd = ::open(path, O_RDONLY);
  if (fd < 0) fail(SC_ERR_IO, std::string("cannot open ") + path);
  const size_t plane = (size_t)w * h * yuv_bytes_per_sample(bit_depth);
  const uint64_t fb = yuv_frame_bytes(w, h, bit_depth);
  for (int f = 0; f < n; ++f) {
    uint8_t* out = static_cast<uint8_t*>(dst) + (size_t)f * plane;
    size_t got = 0;
    const off_t base = (off_t)((uint64_t)(first + f) * fb);
    while (got < plane) {
      const ssize_t r = ::pread(fd, out + got, plane - got, base + (off_t)got);
      if (r <= 0) {
        ::close(fd);
        fail(SC_ERR_IO, std::string("short read on ") + path);
      }
      got += (size_t)r;
    }
  }
  ::close(fd);
}

}  // namespace scb
