// Parameter files in the reference's SSD-PS on-disk format (SURVEY §8(f)
// row 3): what a trained HBM-PS table is exported as, so the reference
// SsdStore (recover/load/fsck/stats) reads it unchanged.
//
// Format (ssd_ps.hpp:50-56), little-endian, one file pf_<id>.bin:
//   header  : "HPSF" | version u16 = 1 | record_count u16 | width u16 |
//             reserved u16                                      (12 B)
//   records : record_count x (key u64 | width x f32 embedding |
//                              width x f32 opt_state)      (8 + 8E B each)
//   footer  : CRC-32 (zlib polynomial) of header + records       (4 B)
// Chunking follows SsdStore::dump (ssd_ps.hpp:229-243): keys in ascending
// order (the std::map order), file_capacity records per file, ids ascending.
#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "tier_internal.h"

using hpsgpu::set_error;

namespace {

constexpr char kMagic[4] = {'H', 'P', 'S', 'F'};
constexpr std::uint16_t kVersion = 1;
constexpr std::size_t kHeader = 12, kFooter = 4;

// CRC-32 (reflected 0xEDB88320, init/final ~0: the zlib crc32 the reference
// links, ssd_ps.hpp:430-440, 516), slicing by 8.
struct Crc32 {
  std::uint32_t t[8][256];
  Crc32() {
    for (std::uint32_t i = 0; i < 256; ++i) {
      std::uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      t[0][i] = c;
    }
    for (std::uint32_t i = 0; i < 256; ++i)
      for (int s = 1; s < 8; ++s) t[s][i] = (t[s - 1][i] >> 8) ^ t[0][t[s - 1][i] & 0xff];
  }
  std::uint32_t update(std::uint32_t crc, const unsigned char* p, std::size_t n) const {
    std::uint32_t c = ~crc;
    while (n >= 8) {
      std::uint32_t lo, hi;
      std::memcpy(&lo, p, 4);
      std::memcpy(&hi, p + 4, 4);
      lo ^= c;
      c = t[7][lo & 0xff] ^ t[6][(lo >> 8) & 0xff] ^ t[5][(lo >> 16) & 0xff] ^ t[4][lo >> 24] ^
          t[3][hi & 0xff] ^ t[2][(hi >> 8) & 0xff] ^ t[1][(hi >> 16) & 0xff] ^ t[0][hi >> 24];
      p += 8;
      n -= 8;
    }
    while (n--) c = t[0][(c ^ *p++) & 0xff] ^ (c >> 8);
    return ~c;
  }
};

const Crc32& crc_table() {
  static const Crc32 c;
  return c;
}

// Host is little-endian x86-64/aarch64, as the format: plain stores.
template <class T>
void put(unsigned char*& p, T v) {
  std::memcpy(p, &v, sizeof v);
  p += sizeof v;
}

template <class T>
T get(const unsigned char* p) {
  T v;
  std::memcpy(&v, p, sizeof v);
  return v;
}

std::string path_of(const char* dir, std::uint64_t id) {
  std::string d(dir);
  if (!d.empty() && d.back() != '/') d += '/';
  return d + "pf_" + std::to_string(id) + ".bin";
}

}  // namespace

extern "C" {

uint32_t hps_crc32(uint32_t crc, const void* data, uint64_t n) {
  return crc_table().update(crc, static_cast<const unsigned char*>(data), n);
}

hps_status hps_pfile_write(const char* dir, const uint64_t* keys, const float* rows,
                           const float* opt_state, uint64_t n, uint32_t width,
                           uint32_t file_capacity, uint64_t first_id, uint64_t* files_out) {
  if (files_out) *files_out = 0;
  if (!dir) return set_error(HPS_ERR_ARG, "store: no directory");
  if (file_capacity < 1 || file_capacity > 0xffff)
    return set_error(HPS_ERR_ARG, "store: file_capacity must be in [1, 65535]");
  if (width < 1 || width > 0xffff) return set_error(HPS_ERR_ARG, "store: bad embedding width");
  if (n == 0) return set_error(HPS_ERR_ARG, "store: dump of empty parameter set");
  if (!keys || !rows) return set_error(HPS_ERR_ARG, "store: null keys/rows");
  for (std::uint64_t i = 1; i < n; ++i)
    if (keys[i] <= keys[i - 1])
      return set_error(HPS_ERR_ARG, "store: keys not strictly ascending at %llu",
                       (unsigned long long)i);
  const std::size_t rec = 8 + 8 * std::size_t(width);
  std::vector<unsigned char> buf;
  std::uint64_t files = 0;
  for (std::uint64_t b = 0; b < n; b += file_capacity, ++files) {
    const std::uint64_t cnt = std::min<std::uint64_t>(file_capacity, n - b);
    buf.resize(kHeader + cnt * rec + kFooter);
    unsigned char* p = buf.data();
    std::memcpy(p, kMagic, 4);
    p += 4;
    put<std::uint16_t>(p, kVersion);
    put<std::uint16_t>(p, std::uint16_t(cnt));
    put<std::uint16_t>(p, std::uint16_t(width));
    put<std::uint16_t>(p, 0);
    for (std::uint64_t i = b; i < b + cnt; ++i) {
      put<std::uint64_t>(p, keys[i]);
      std::memcpy(p, rows + i * width, 4 * std::size_t(width));
      p += 4 * std::size_t(width);
      if (opt_state)
        std::memcpy(p, opt_state + i * width, 4 * std::size_t(width));
      else
        std::memset(p, 0, 4 * std::size_t(width));  // SparseParam(width) (types.hpp:36)
      p += 4 * std::size_t(width);
    }
    put<std::uint32_t>(p, hps_crc32(0, buf.data(), std::uint64_t(p - buf.data())));
    // a temp name, then rename: recover() (ssd_ps.hpp:362-369) only maps
    // pf_<id>.bin, so an interrupted export leaves no half-written file
    const std::string fin = path_of(dir, first_id + files), tmp = fin + ".tmp";
    std::FILE* f = std::fopen(tmp.c_str(), "wb");
    if (!f) return set_error(HPS_ERR_ARG, "store: cannot create %s: %s", tmp.c_str(),
                             std::strerror(errno));
    const bool ok = std::fwrite(buf.data(), 1, buf.size(), f) == buf.size();
    if (std::fclose(f) != 0 || !ok) {
      std::remove(tmp.c_str());
      return set_error(HPS_ERR_ARG, "store: short write (disk full?)");
    }
    if (std::rename(tmp.c_str(), fin.c_str()) != 0)
      return set_error(HPS_ERR_ARG, "store: cannot rename %s: %s", tmp.c_str(),
                       std::strerror(errno));
  }
  if (files_out) *files_out = files;
  return HPS_OK;
}

hps_status hps_pfile_read(const char* path, uint64_t* keys, float* rows, float* opt_state,
                          uint64_t cap, uint64_t* n_out, uint32_t* width_out) {
  if (!path) return set_error(HPS_ERR_ARG, "store: no path");
  std::FILE* f = std::fopen(path, "rb");
  if (!f) return set_error(HPS_ERR_CORRUPT, "store: mapped file absent: %s", path);
  std::vector<unsigned char> buf;
  unsigned char chunk[1 << 16];
  std::size_t got;
  while ((got = std::fread(chunk, 1, sizeof chunk, f)) > 0) buf.insert(buf.end(), chunk, chunk + got);
  std::fclose(f);
  // the checks and messages of SsdStore::read_file_at (ssd_ps.hpp:495-520)
  if (buf.size() < kHeader + kFooter)
    return set_error(HPS_ERR_CORRUPT, "store: truncated file %s", path);
  if (std::memcmp(buf.data(), kMagic, 4) != 0)
    return set_error(HPS_ERR_CORRUPT, "store: bad magic in %s", path);
  if (get<std::uint16_t>(buf.data() + 4) != kVersion)
    return set_error(HPS_ERR_CORRUPT, "store: bad version in %s", path);
  const std::size_t count = get<std::uint16_t>(buf.data() + 6);
  const std::size_t width = get<std::uint16_t>(buf.data() + 8);
  if (width_out && *width_out != 0 && *width_out != width)
    return set_error(HPS_ERR_CORRUPT, "store: embedding width mismatch in %s", path);
  if (buf.size() != kHeader + count * (8 + 8 * width) + kFooter)
    return set_error(HPS_ERR_CORRUPT, "store: size mismatch in %s", path);
  const std::size_t payload = buf.size() - kFooter;
  if (get<std::uint32_t>(buf.data() + payload) != hps_crc32(0, buf.data(), payload))
    return set_error(HPS_ERR_CORRUPT, "store: checksum mismatch in %s", path);
  if (n_out) *n_out = count;
  if (width_out) *width_out = std::uint32_t(width);
  if (!keys && !rows && !opt_state) return HPS_OK;  // sizing call
  if (count > cap) return set_error(HPS_ERR_CAPACITY, "store: %zu records > cap %llu", count,
                                    (unsigned long long)cap);
  const unsigned char* p = buf.data() + kHeader;
  for (std::size_t i = 0; i < count; ++i) {
    if (keys) keys[i] = get<std::uint64_t>(p);
    p += 8;
    if (rows) std::memcpy(rows + i * width, p, 4 * width);
    p += 4 * width;
    if (opt_state) std::memcpy(opt_state + i * width, p, 4 * width);
    p += 4 * width;
  }
  return HPS_OK;
}

hps_status hps_export(hps_tier_t h, const char* dir, uint32_t file_capacity, uint64_t first_id,
                      uint64_t* files_out) {
  if (files_out) *files_out = 0;
  std::uint64_t cap = 0, occ = 0, width = 0;
  hps_status st = hps_table_info(h, &cap, &occ, &width);
  if (st != HPS_OK) return st;
  std::uint64_t rw = 0;
  st = hps_row_width(h, &rw);
  if (st != HPS_OK) return st;
  std::vector<std::uint64_t> keys(occ);
  std::vector<float> rows(occ * rw);
  std::uint64_t n = 0;
  st = hps_dump(h, keys.data(), rows.data(), &n);
  if (st != HPS_OK) return st;
  if (rw == width)  // SGD: no optimizer state in the row (opt_state written as zeros)
    return hps_pfile_write(dir, keys.data(), rows.data(), nullptr, n, std::uint32_t(width),
                           file_capacity, first_id, files_out);
  // Adagrad: each row is the embedding then its accumulator, the record's
  // embedding and opt_state (types.hpp:30-39, ssd_ps.hpp:50-56)
  std::vector<float> emb(n * width), opt(n * width);
  for (std::uint64_t i = 0; i < n; ++i) {
    std::memcpy(&emb[i * width], &rows[i * rw], width * 4);
    std::memcpy(&opt[i * width], &rows[i * rw + width], width * 4);
  }
  return hps_pfile_write(dir, keys.data(), emb.data(), opt.data(), n, std::uint32_t(width),
                         file_capacity, first_id, files_out);
}

}  // extern "C"
