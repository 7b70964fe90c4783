// AVDB vector files (reference vfs.py, docs/file-format.md) -> GPU KV slabs.
//
// Host side (no device needed): header + directory-chain parsing
// (read_header / read_directory, vfs.py:247-286), and the writer
// (write_vector_file, vfs.py:188-244), byte-identical to the reference's for
// vector-only files (fp32, or fp16 narrowed round-to-nearest-even).
//
// Load path (read_vector_file, vfs.py:289-338, as ContextStore._load_existing
// uses it, store.py:569-609): each file image is pread into a caller-owned
// PINNED host buffer, and ONE kernel per call walks the data blocks in
// directory order straight out of pinned memory (zero-copy over PCIe, no
// device staging copy, no numpy) and writes the [n][dim] rows of every file
// into the device slab, widening fp16 or narrowing to bf16 on the way.
#include <fcntl.h>
#include <unistd.h>

#include <cstring>
#include <vector>

#include "alaya_dispatch.cuh"

namespace alaya {
namespace {

constexpr uint32_t kBlock = 4096;
constexpr uint32_t kBlockHdr = 16;
constexpr uint32_t kPayload = kBlock - kBlockHdr;
constexpr uint32_t kDirPrefix = 16;  // prev u64, count u32, pad 4
constexpr uint32_t kDirEntry = 16;   // offset u64, type u8, pad 3, count u32
constexpr uint32_t kDirCap = (kPayload - kDirPrefix) / kDirEntry;
enum : uint8_t { kIndex = 1, kData = 2, kDirectory = 3, kTombstone = 4 };

template <typename T>
T rd(const uint8_t* p) {
  T v;
  memcpy(&v, p, sizeof(T));
  return v;
}
template <typename T>
void wr(uint8_t* p, T v) {
  memcpy(p, &v, sizeof(T));
}

struct Dir {
  uint64_t offset;
  uint8_t type;
  uint32_t count;
};

int read_exact(int fd, uint64_t off, void* dst, size_t n, const char* path) {
  size_t got = 0;
  while (got < n) {
    const ssize_t r = pread(fd, static_cast<char*>(dst) + got, n - got, (off_t)(off + got));
    if (r <= 0) return fail(ALAYA_ERR_ARG, "%s @ %llu: short read", path, (unsigned long long)(off + got));
    got += (size_t)r;
  }
  return ALAYA_OK;
}

// header + directory of one file (read_header / read_directory)
int parse(const char* path, alaya_avdb_info* info, std::vector<Dir>* dir) {
  const int fd = open(path, O_RDONLY);
  if (fd < 0) return fail(ALAYA_ERR_ARG, "%s: cannot open", path);
  uint8_t blk[kBlock];
  int rc = read_exact(fd, 0, blk, kBlock, path);
  if (rc) { close(fd); return rc; }
  if (memcmp(blk, "AVDB", 4) != 0) { close(fd); return fail(ALAYA_ERR_ARG, "%s @ 0: bad magic", path); }
  const uint32_t version = rd<uint32_t>(blk + 4), dim = rd<uint32_t>(blk + 8);
  const uint64_t n = rd<uint64_t>(blk + 12);
  const uint32_t width = rd<uint32_t>(blk + 20), bsz = rd<uint32_t>(blk + 24);
  const uint64_t dir_off = rd<uint64_t>(blk + 28), index_head = rd<uint64_t>(blk + 36);
  if (version != 1) { close(fd); return fail(ALAYA_ERR_ARG, "%s @ 0: unsupported version %u", path, version); }
  if (bsz != kBlock) { close(fd); return fail(ALAYA_ERR_ARG, "%s @ 0: unsupported block size %u", path, bsz); }
  if (width != 16 && width != 32) { close(fd); return fail(ALAYA_ERR_ARG, "%s: element width %u", path, width); }
  const off_t end = lseek(fd, 0, SEEK_END);
  std::vector<std::vector<Dir>> chains;
  uint64_t off = dir_off;
  for (int guard = 0;; ++guard) {
    if (off % kBlock || off + kBlock > (uint64_t)end || guard > (1 << 20)) {
      close(fd);
      return fail(ALAYA_ERR_ARG, "%s @ %llu: bad directory offset", path, (unsigned long long)off);
    }
    if ((rc = read_exact(fd, off, blk, kBlock, path))) { close(fd); return rc; }
    if (blk[0] != kDirectory) {
      close(fd);
      return fail(ALAYA_ERR_ARG, "%s @ %llu: expected directory block, found %u", path,
                  (unsigned long long)off, blk[0]);
    }
    const uint8_t* pl = blk + kBlockHdr;
    const uint64_t prev = rd<uint64_t>(pl);
    const uint32_t cnt = rd<uint32_t>(pl + 8);
    if (cnt > kDirCap) { close(fd); return fail(ALAYA_ERR_ARG, "%s: directory overflow", path); }
    std::vector<Dir> ch(cnt);
    for (uint32_t i = 0; i < cnt; ++i) {
      const uint8_t* e = pl + kDirPrefix + i * kDirEntry;
      ch[i] = {rd<uint64_t>(e), e[8], rd<uint32_t>(e + 12)};
    }
    chains.push_back(std::move(ch));
    if (prev == 0) break;
    off = prev;
  }
  close(fd);
  dir->clear();
  for (auto it = chains.rbegin(); it != chains.rend(); ++it) dir->insert(dir->end(), it->begin(), it->end());
  uint64_t rows = 0;
  uint32_t ndata = 0, ntomb = 0, nindex = 0;
  for (const Dir& d : *dir) {
    if (d.offset % kBlock || d.offset + kBlock > (uint64_t)end)
      return fail(ALAYA_ERR_ARG, "%s @ %llu: block outside the file", path, (unsigned long long)d.offset);
    if (d.type == kData) { rows += d.count; ++ndata; }
    else if (d.type == kTombstone) ntomb += d.count;
    else if (d.type == kIndex) ++nindex;
    else return fail(ALAYA_ERR_ARG, "%s @ %llu: unexpected block type %u in directory", path,
                     (unsigned long long)d.offset, d.type);
  }
  if (rows != n)
    return fail(ALAYA_ERR_ARG, "%s @ 0: expected %llu vectors, found %llu", path, (unsigned long long)n,
                (unsigned long long)rows);
  const uint32_t slot = dim * width / 8;
  for (const Dir& d : *dir)
    if (d.type == kData && (uint64_t)d.count * slot > kPayload)
      return fail(ALAYA_ERR_ARG, "%s @ %llu: data block overflows", path, (unsigned long long)d.offset);
  info->dim = dim;
  info->element_width = width;
  info->n_vectors = n;
  info->n_data_blocks = ndata;
  info->n_index_blocks = nindex;
  info->n_tombstones = ntomb;
  info->file_bytes = (uint64_t)end;
  info->directory_offset = dir_off;
  info->index_head = index_head;
  return ALAYA_OK;
}

// float32 -> IEEE half, round to nearest even (numpy astype(float16))
uint16_t to_half(float f) {
  uint32_t x;
  memcpy(&x, &f, 4);
  const uint32_t sign = (x >> 16) & 0x8000u;
  const uint32_t absx = x & 0x7fffffffu;
  if (absx >= 0x7f800000u) return (uint16_t)(sign | 0x7c00u | (absx > 0x7f800000u ? 0x200u : 0u));
  if (absx >= 0x477ff000u) return (uint16_t)(sign | 0x7c00u);  // rounds to >= 65520: inf
  if (absx < 0x38800000u) {  // subnormal half (or zero)
    if (absx < 0x33000000u) return (uint16_t)sign;  // < 2^-25: rounds to zero
    const uint32_t e = absx >> 23;
    const uint32_t m = (absx & 0x7fffffu) | 0x800000u;
    const int shift = 126 - (int)e;  // 14..24
    uint32_t r = m >> shift;
    const uint32_t rem = m & ((1u << shift) - 1u), half = 1u << (shift - 1);
    if (rem > half || (rem == half && (r & 1u))) ++r;
    return (uint16_t)(sign | r);
  }
  uint32_t r = ((absx >> 13) - (112u << 10));
  const uint32_t rem = absx & 0x1fffu;
  if (rem > 0x1000u || (rem == 0x1000u && (r & 1u))) ++r;
  return (uint16_t)(sign | r);
}

struct BlockJob {
  const uint8_t* src;  // pinned host (UVA) address of the block payload
  int64_t row0;        // first destination row (within the file)
  int32_t count;
  int32_t file;
};

__device__ __forceinline__ float half_to_float(uint16_t h) { return __half2float(__ushort_as_half(h)); }

// One CTA per data block: rows of `count` slots from pinned host memory into
// dst[file * file_stride + (row0 + r) * dim].
template <typename TO>
__global__ void __launch_bounds__(256)
    avdb_unpack_kernel(const BlockJob* __restrict__ jobs, int width, int dim, TO* __restrict__ dst,
                       int64_t file_stride) {
  const BlockJob j = jobs[blockIdx.x];
  const int64_t total = (int64_t)j.count * dim;
  TO* out = dst + (size_t)j.file * file_stride + (size_t)j.row0 * dim;
  for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
    float x;
    if (width == 32) x = reinterpret_cast<const float*>(j.src)[e];
    else x = half_to_float(reinterpret_cast<const uint16_t*>(j.src)[e]);
    if constexpr (std::is_same_v<TO, float>) out[e] = x;
    else out[e] = __float2bfloat16_rn(x);
  }
}

}  // namespace
}  // namespace alaya

using namespace alaya;

extern "C" {

int alaya_avdb_stat(const char* path, alaya_avdb_info* out) {
  if (!path || !out) return fail(ALAYA_ERR_ARG, "null path/info");
  std::vector<Dir> dir;
  return parse(path, out, &dir);
}

int alaya_avdb_write(const char* path, const float* vectors, int64_t n, int dim, int element_width) {
  if (!path || (n > 0 && !vectors) || n < 0 || dim < 1) return fail(ALAYA_ERR_ARG, "bad avdb write arguments");
  if (element_width != 16 && element_width != 32)
    return fail(ALAYA_ERR_ARG, "unsupported element width %d", element_width);
  const uint32_t slot = (uint32_t)dim * element_width / 8;
  const uint32_t per = kPayload / slot;
  if (per < 1) return fail(ALAYA_ERR_ARG, "vector slot of %u bytes does not fit in a block", slot);
  const uint64_t ndata = n ? (uint64_t)(n + per - 1) / per : 0;
  std::vector<Dir> entries;
  std::vector<uint8_t> img((size_t)kBlock * (1 + ndata), 0);
  uint64_t off = kBlock;
  for (uint64_t bidx = 0; bidx < ndata; ++bidx) {
    const int64_t lo = (int64_t)(bidx * per);
    const uint32_t count = (uint32_t)std::min<int64_t>(per, n - lo);
    uint8_t* b = img.data() + off;
    b[0] = kData;
    wr<uint32_t>(b + 4, count * slot);
    uint8_t* pl = b + kBlockHdr;
    const float* src = vectors + (size_t)lo * dim;
    if (element_width == 32) {
      memcpy(pl, src, (size_t)count * slot);
    } else {
      for (size_t e = 0; e < (size_t)count * dim; ++e) wr<uint16_t>(pl + 2 * e, to_half(src[e]));
    }
    entries.push_back({off, kData, count});
    off += kBlock;
  }
  // directory chain (vfs.py:168-185): chunks of kDirCap, each pointing back
  size_t nchunks = entries.empty() ? 1 : (entries.size() + kDirCap - 1) / kDirCap;
  uint64_t prev = 0, dir_off = off;
  img.resize((size_t)off + (size_t)nchunks * kBlock, 0);
  for (size_t c = 0; c < nchunks; ++c) {
    const size_t a = c * kDirCap, e = std::min(entries.size(), a + kDirCap);
    uint8_t* b = img.data() + off;
    b[0] = kDirectory;
    wr<uint32_t>(b + 4, kDirPrefix + (uint32_t)(e - a) * kDirEntry);
    uint8_t* pl = b + kBlockHdr;
    wr<uint64_t>(pl, prev);
    wr<uint32_t>(pl + 8, (uint32_t)(e - a));
    for (size_t i = a; i < e; ++i) {
      uint8_t* q = pl + kDirPrefix + (i - a) * kDirEntry;
      wr<uint64_t>(q, entries[i].offset);
      q[8] = entries[i].type;
      wr<uint32_t>(q + 12, entries[i].count);
    }
    prev = off;
    dir_off = off;
    off += kBlock;
  }
  uint8_t* h = img.data();
  memcpy(h, "AVDB", 4);
  wr<uint32_t>(h + 4, 1u);
  wr<uint32_t>(h + 8, (uint32_t)dim);
  wr<uint64_t>(h + 12, (uint64_t)n);
  wr<uint32_t>(h + 20, (uint32_t)element_width);
  wr<uint32_t>(h + 24, kBlock);
  wr<uint64_t>(h + 28, dir_off);
  wr<uint64_t>(h + 36, 0ull);
  const int fd = open(path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
  if (fd < 0) return fail(ALAYA_ERR_ARG, "%s @ 0: write failed (open)", path);
  size_t put = 0;
  while (put < img.size()) {
    const ssize_t w = write(fd, img.data() + put, img.size() - put);
    if (w <= 0) { close(fd); return fail(ALAYA_ERR_ARG, "%s @ %zu: write failed", path, put); }
    put += (size_t)w;
  }
  close(fd);
  return ALAYA_OK;
}

int alaya_avdb_graph(const char* path, int64_t* n_nodes, int64_t* n_edges, int32_t* entry_point,
                     int32_t* max_degree, int32_t* degrees, int32_t* nbrs) {
  if (!path || !n_nodes || !n_edges || !entry_point || !max_degree) return fail(ALAYA_ERR_ARG, "null outputs");
  alaya_avdb_info info;
  std::vector<Dir> dir;
  int rc = parse(path, &info, &dir);
  if (rc) return rc;
  *n_nodes = *n_edges = 0;
  *entry_point = *max_degree = 0;
  if (info.n_index_blocks == 0) return ALAYA_OK;
  // the index chain's logical stream (vfs.py:126-145, index blocks in directory order)
  std::vector<uint8_t> stream;
  const int fd = open(path, O_RDONLY);
  if (fd < 0) return fail(ALAYA_ERR_ARG, "%s: cannot open", path);
  uint8_t blk[kBlock];
  for (const Dir& d : dir) {
    if (d.type != kIndex) continue;
    if ((rc = read_exact(fd, d.offset, blk, kBlock, path))) { close(fd); return rc; }
    const uint32_t len = rd<uint32_t>(blk + 4);
    if (blk[0] != kIndex || len > kPayload) { close(fd); return fail(ALAYA_ERR_ARG, "%s @ %llu: bad index block", path, (unsigned long long)d.offset); }
    stream.insert(stream.end(), blk + kBlockHdr, blk + kBlockHdr + len);
  }
  close(fd);
  if (stream.size() < 12) return fail(ALAYA_ERR_ARG, "%s: truncated index stream", path);
  const uint32_t ep = rd<uint32_t>(stream.data()), md = rd<uint32_t>(stream.data() + 4);
  const uint32_t nn = rd<uint32_t>(stream.data() + 8);
  if (stream.size() < 12 + 4ull * nn) return fail(ALAYA_ERR_ARG, "%s: truncated degree table", path);
  uint64_t ne = 0;
  for (uint32_t i = 0; i < nn; ++i) ne += rd<uint32_t>(stream.data() + 12 + 4ull * i);
  if (stream.size() < 12 + 4ull * nn + 4ull * ne) return fail(ALAYA_ERR_ARG, "%s: truncated neighbour list", path);
  *n_nodes = nn;
  *n_edges = (int64_t)ne;
  *entry_point = (int32_t)ep;
  *max_degree = (int32_t)md;
  if (degrees) memcpy(degrees, stream.data() + 12, 4ull * nn);
  if (nbrs) {
    const uint8_t* fl = stream.data() + 12 + 4ull * nn;
    for (uint64_t e = 0; e < ne; ++e) {
      const uint32_t v = rd<uint32_t>(fl + 4 * e);
      if (v >= info.n_vectors) return fail(ALAYA_ERR_ARG, "%s @ 0: node references a missing vector slot", path);
      nbrs[e] = (int32_t)v;
    }
  }
  return ALAYA_OK;
}

size_t alaya_avdb_staging_bytes(const char* const* paths, int n_files) {
  size_t tot = 0;
  for (int i = 0; i < n_files; ++i) {
    alaya_avdb_info info;
    std::vector<Dir> dir;
    if (!paths || !paths[i] || parse(paths[i], &info, &dir)) return 0;
    tot += (size_t)info.file_bytes + 256 + (size_t)info.n_data_blocks * sizeof(BlockJob);
  }
  return tot + 256;
}

int alaya_avdb_load(const char* const* paths, int n_files, int64_t n, int dim, int dst_dtype,
                    void* d_dst, int64_t dst_file_stride, void* h_staging, size_t staging_bytes,
                    void* stream) {
  if (!paths || n_files < 1 || !d_dst || !h_staging || dim < 1 || n < 0)
    return fail(ALAYA_ERR_ARG, "bad avdb load arguments");
  if (dst_dtype != ALAYA_F32 && dst_dtype != ALAYA_BF16) return fail(ALAYA_ERR_ARG, "bad dtype");
  if (dst_file_stride < n * dim) return fail(ALAYA_ERR_SHAPE, "dst_file_stride too small");
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, h_staging) != cudaSuccess || attr.type != cudaMemoryTypeHost)
    return fail(ALAYA_ERR_ARG, "staging buffer must be pinned host memory (cudaHostAlloc / pin_memory)");
  // file images, then the block-job table, in the staging buffer
  std::vector<BlockJob> jobs;
  std::vector<alaya_avdb_info> infos((size_t)n_files);
  uint8_t* base = static_cast<uint8_t*>(h_staging);
  size_t used = 0;
  int width = 0;
  for (int f = 0; f < n_files; ++f) {
    std::vector<Dir> dir;
    int rc = parse(paths[f], &infos[f], &dir);
    if (rc) return rc;
    const alaya_avdb_info& in = infos[f];
    if ((int64_t)in.n_vectors != n || (int)in.dim != dim)
      return fail(ALAYA_ERR_SHAPE, "%s: %llu x %u vectors, expected %lld x %d", paths[f],
                  (unsigned long long)in.n_vectors, in.dim, (long long)n, dim);
    if (width && (int)in.element_width != width)
      return fail(ALAYA_ERR_ARG, "%s: mixed element widths in one load", paths[f]);
    width = (int)in.element_width;
    used = (used + 255) & ~(size_t)255;
    if (used + in.file_bytes > staging_bytes)
      return fail(ALAYA_ERR_WORKSPACE, "staging buffer %zu bytes too small", staging_bytes);
    const int fd = open(paths[f], O_RDONLY);
    if (fd < 0) return fail(ALAYA_ERR_ARG, "%s: cannot open", paths[f]);
    rc = read_exact(fd, 0, base + used, (size_t)in.file_bytes, paths[f]);
    close(fd);
    if (rc) return rc;
    int64_t row = 0;
    for (const Dir& d : dir) {
      if (d.type != kData || d.count == 0) continue;
      const uint8_t* b = base + used + d.offset;
      if (b[0] != kData) return fail(ALAYA_ERR_ARG, "%s @ %llu: directory/block type mismatch", paths[f],
                                     (unsigned long long)d.offset);
      jobs.push_back({b + kBlockHdr, row, (int32_t)d.count, f});
      row += d.count;
    }
    used += (size_t)in.file_bytes;
  }
  if (jobs.empty()) return ALAYA_OK;
  used = (used + 255) & ~(size_t)255;
  const size_t jb = jobs.size() * sizeof(BlockJob);
  if (used + jb > staging_bytes) return fail(ALAYA_ERR_WORKSPACE, "staging buffer %zu bytes too small", staging_bytes);
  BlockJob* tab = reinterpret_cast<BlockJob*>(base + used);
  memcpy(tab, jobs.data(), jb);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const unsigned grid = (unsigned)jobs.size();
  if (dst_dtype == ALAYA_F32)
    avdb_unpack_kernel<float><<<grid, 256, 0, st>>>(tab, width, dim, static_cast<float*>(d_dst), dst_file_stride);
  else
    avdb_unpack_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(tab, width, dim, static_cast<__nv_bfloat16*>(d_dst),
                                                            dst_file_stride);
  return cuda_check("avdb_unpack_kernel");
}

}  // extern "C"
