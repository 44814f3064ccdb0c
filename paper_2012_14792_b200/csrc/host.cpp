// Host-side pieces of the reference API behind the C-ABI: the CTU-complexity
// model (cost.cpp:40-95), the TextureStats tables and SliceMoments::sse
// (texture.cpp:83-130), PrefixSumTable (cost.cpp:97-112) and split_even
// (grid.cpp:52-60).  All O(cells) bookkeeping that the reference also keeps
// on the host; the per-candidate work runs in the sm_100a kernels.  These
// functions let a C++ or Python binding provide the whole partitioner API
// from libslicecraft_b200.so alone (dropin/slicecraft_api.cpp).
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "slicecraft_b200.h"

namespace scb {
sc_status set_last_error(sc_status s, const char* msg);  // api.cu (sc_last_error)
}

namespace {

struct HostFail {
  sc_status status;
  std::string msg;
};
[[noreturn]] void hfail(sc_status s, const std::string& m) { throw HostFail{s, m}; }

template <typename F>
sc_status host_guarded(F&& fn) {
  try {
    fn();
    return scb::set_last_error(SC_OK, "");
  } catch (const HostFail& f) {
    return scb::set_last_error(f.status, f.msg.c_str());
  } catch (const std::exception& e) {
    return scb::set_last_error(SC_ERR_INTERNAL, e.what());
  }
}

bool same_grid(const sc_grid& a, const sc_grid& b) {
  return a.frame_width == b.frame_width && a.frame_height == b.frame_height &&
         a.ctu_size == b.ctu_size && a.cols == b.cols && a.rows == b.rows;
}

// temporal_layer_of_poc (cost.cpp:28-38)
int temporal_layer(int poc, int gop) {
  if (gop < 1 || (gop & (gop - 1)) != 0)
    hfail(SC_ERR_CONFIG, "gop size must be a power of two, got " + std::to_string(gop));
  if (poc < 0) hfail(SC_ERR_CONFIG, "poc must be >= 0");
  const unsigned rem = (unsigned)poc % (unsigned)gop;
  return rem == 0 ? 0 : __builtin_ctz((unsigned)gop) - __builtin_ctz(rem);
}

int64_t cell_pixels(const sc_grid& g, int x, int y) {
  const int w = g.frame_width - x * g.ctu_size, h = g.frame_height - y * g.ctu_size;
  return (int64_t)(w < g.ctu_size ? w : g.ctu_size) * (h < g.ctu_size ? h : g.ctu_size);
}

}  // namespace

extern "C" {

sc_status sc_cost_map_check(const sc_grid* history_grid, const sc_grid* map_grid,
                            const double* times, int64_t n_times, int32_t poc,
                            const int32_t* history_pocs, int32_t n_history) {
  return host_guarded([&] {
    if (!history_grid || !map_grid || (n_times > 0 && !times) ||
        (n_history > 0 && !history_pocs))
      hfail(SC_ERR_USAGE, "NULL argument");
    // CostHistory::append (cost.cpp:45-64): grid, entry count, values, poc
    if (!same_grid(*history_grid, *map_grid))
      hfail(SC_ERR_GEOMETRY, "cost map grid does not match the history grid");
    if (n_times != (int64_t)history_grid->cols * history_grid->rows)
      hfail(SC_ERR_GEOMETRY, "cost map has wrong number of entries");
    for (int64_t i = 0; i < n_times; ++i)
      if (!std::isfinite(times[i]) || times[i] < 0.0)
        hfail(SC_ERR_FORMAT, "CTU times must be finite and >= 0");
    for (int32_t i = 0; i < n_history; ++i)
      if (history_pocs[i] == poc)
        hfail(SC_ERR_TRACE, "duplicate poc " + std::to_string(poc) + " in cost history");
  });
}

sc_status sc_estimate_ctu_times(const sc_grid* grid, int32_t gop_size, int32_t n_maps,
                                const double* const* maps, const int32_t* pocs,
                                const int32_t* temporal_layers, int32_t poc, double* out,
                                int32_t* source, int32_t* source_poc, int32_t* out_layer) {
  return host_guarded([&] {
    if (!grid || !out || (n_maps > 0 && (!maps || !pocs || !temporal_layers)))
      hfail(SC_ERR_USAGE, "NULL argument");
    // estimate_ctu_times (cost.cpp:66-95): the most recent map of the same
    // temporal layer, else the most recent map, else all-ones
    const int tl = temporal_layer(poc, gop_size);
    const size_t cells = (size_t)grid->cols * grid->rows;
    int pick = -1, src = SC_SOURCE_UNIFORM;
    for (int i = n_maps - 1; i >= 0; --i)
      if (temporal_layers[i] == tl) {
        pick = i;
        src = SC_SOURCE_CO_TEMPORAL_LAYER;
        break;
      }
    if (pick < 0 && n_maps > 0) {
      pick = n_maps - 1;
      src = SC_SOURCE_MOST_RECENT_ANY;
    }
    if (pick >= 0) {
      if (!maps[pick]) hfail(SC_ERR_USAGE, "NULL cost map");
      std::memcpy(out, maps[pick], cells * sizeof(double));
    } else {
      for (size_t i = 0; i < cells; ++i) out[i] = 1.0;
    }
    if (source) *source = src;
    if (source_poc) *source_poc = pick >= 0 ? pocs[pick] : -1;
    if (out_layer) *out_layer = tl;
  });
}

sc_status sc_texture_tables(const sc_grid* grid, const sc_ctu_record* records, int64_t n_records,
                            uint64_t* pre_count, uint64_t* pre_sum, uint64_t* pre_sumsq) {
  return host_guarded([&] {
    if (!grid || (n_records > 0 && !records)) hfail(SC_ERR_USAGE, "NULL argument");
    const sc_grid& g = *grid;
    // TextureStats ctor (texture.cpp:90-111): record count, pixel counts,
    // count*sumsq >= sum^2 in 128-bit integers
    if (n_records != (int64_t)g.cols * g.rows)
      hfail(SC_ERR_GEOMETRY, "record count " + std::to_string(n_records) +
                                 " does not match grid cell count " +
                                 std::to_string((int64_t)g.cols * g.rows));
    for (int y = 0; y < g.rows; ++y)
      for (int x = 0; x < g.cols; ++x) {
        const sc_ctu_record& r = records[(size_t)y * g.cols + x];
        if (r.count != (uint64_t)cell_pixels(g, x, y))
          hfail(SC_ERR_FORMAT, "CTU pixel count mismatch at (" + std::to_string(x) + "," +
                                   std::to_string(y) + ")");
        if ((unsigned __int128)r.count * r.sumsq < (unsigned __int128)r.sum * r.sum)
          hfail(SC_ERR_FORMAT, "CTU statistics violate count*sumsq >= sum^2 at (" +
                                   std::to_string(x) + "," + std::to_string(y) + ")");
      }
    // (cols+1) x (rows+1) inclusion-exclusion tables, modular u64
    // (texture.cpp:113-129); any of the outputs may be NULL
    const size_t stride = (size_t)g.cols + 1, n = stride * ((size_t)g.rows + 1);
    uint64_t* tab[3] = {pre_count, pre_sum, pre_sumsq};
    for (int k = 0; k < 3; ++k) {
      uint64_t* t = tab[k];
      if (!t) continue;
      std::memset(t, 0, n * sizeof(uint64_t));
      for (int y = 0; y < g.rows; ++y)
        for (size_t x = 0; x < (size_t)g.cols; ++x) {
          const sc_ctu_record& r = records[(size_t)y * g.cols + x];
          const uint64_t v = k == 0 ? r.count : (k == 1 ? r.sum : r.sumsq);
          const size_t i = (size_t)(y + 1) * stride + x + 1;
          t[i] = v + t[i - 1] + t[i - stride] - t[i - stride - 1];
        }
    }
  });
}

sc_status sc_moments_sse(const sc_ctu_record* m, double* out) {
  return host_guarded([&] {
    if (!m || !out) hfail(SC_ERR_USAGE, "NULL argument");
    // SliceMoments::sse (texture.cpp:83-88): exact signed 128-bit numerator,
    // converted to double (round to nearest even), then one division
    if (m->count == 0) {
      *out = 0.0;
      return;
    }
    const __int128 num = (__int128)m->count * (__int128)m->sumsq - (__int128)m->sum * (__int128)m->sum;
    *out = (double)num / (double)m->count;
  });
}

sc_status sc_prefix_sum_table(const double* values, int64_t n_values, int32_t cols, int32_t rows,
                              double* table) {
  return host_guarded([&] {
    if ((n_values > 0 && !values) || !table) hfail(SC_ERR_USAGE, "NULL argument");
    if (cols < 0 || rows < 0 || n_values != (int64_t)cols * rows)
      hfail(SC_ERR_GEOMETRY, "value count does not match table dimensions");
    // PrefixSumTable (cost.cpp:97-112): ((v + left) + up) - up_left, row-major
    const size_t stride = (size_t)cols + 1;
    std::memset(table, 0, stride * ((size_t)rows + 1) * sizeof(double));
    for (int y = 0; y < rows; ++y)
      for (int x = 0; x < cols; ++x) {
        const size_t i = (size_t)(y + 1) * stride + (size_t)x + 1;
        table[i] = values[(size_t)y * cols + x] + table[i - 1] + table[i - stride] -
                   table[i - stride - 1];
      }
  });
}

sc_status sc_split_even(int32_t total, int32_t parts, int32_t* out) {
  return host_guarded([&] {
    if (!out) hfail(SC_ERR_USAGE, "NULL argument");
    if (parts < 1 || parts > total) hfail(SC_ERR_USAGE, "split_even needs 1 <= parts <= total");
    // grid.cpp:52-60: near-equal parts, the larger ones first
    for (int i = 0; i < parts; ++i) out[i] = total / parts + (i < total % parts ? 1 : 0);
  });
}

}  // extern "C"
