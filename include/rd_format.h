/*
 * rd_format.h — the on-disk index format shared by both implementations of rd.h
 * (the B200 engine and the CPU oracle), so a file written by one loads in the other.
 *
 * SURVEY.md §8f row 3 ("on-disk index format + loader"): the reference's knowledge
 * base is a set of fixed-size partitions on disk (DatabaseProfile::partition_bytes,
 * /root/reference/proj/core/include/ragsim/domain.hpp:57-68; 32 x 8 GiB in
 * proj/configs/default_8b.json:20-25) whose load cost is partition_bytes / bw_cpu_disk
 * (core/src/domain.cpp:48-50). Here a partition is an inverted list and the file holds
 * every list contiguously in list order, so loading one list is one contiguous read.
 *
 * Layout (little-endian; every section starts on a 4096-byte boundary):
 *   header  (4096 B)  rd_file_header below, zero padded
 *   list_offsets      int64[nlist + 1]      prefix row offsets, 0 .. n
 *   ids               int64[n]              user id of each row
 *   centroids         float32[nlist * d]
 *   vectors           float32[n * d]        row-major, list order
 * `check` is FNV-1a 64 over the header bytes before it followed by the list_offsets
 * section; a mismatch, a wrong magic/version or inconsistent sizes is a parse error
 * (RD_ERR_INVALID, the ragsim ParseError exit code 2).
 * Residency is not stored: a loaded index is fully resident until rd_index_place.
 */
#ifndef RD_FORMAT_H_
#define RD_FORMAT_H_

#include <stddef.h>
#include <stdint.h>
#include <string.h>

#define RD_FILE_MAGIC "RDIDX\0v1"
#define RD_FILE_VERSION 1u
#define RD_FILE_ALIGN 4096ull

typedef struct {
  char magic[8];
  uint32_t version;
  uint32_t flags;
  int64_t n;
  int32_t d;
  int32_t nlist;
  uint64_t off_list_offsets;
  uint64_t off_ids;
  uint64_t off_centroids;
  uint64_t off_vectors;
  uint64_t file_bytes;
  uint64_t check;
} rd_file_header;

static inline uint64_t rd_fmt_align(uint64_t x) { return (x + RD_FILE_ALIGN - 1) & ~(RD_FILE_ALIGN - 1); }

static inline uint64_t rd_fmt_fnv1a(uint64_t h, const void* p, uint64_t len) {
  const unsigned char* b = (const unsigned char*)p;
  for (uint64_t i = 0; i < len; ++i) {
    h ^= b[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

/* Fills the section layout for (n, d, nlist); the writer then sets check = rd_fmt_check(). */
static inline void rd_fmt_layout(rd_file_header* h, int64_t n, int32_t d, int32_t nlist) {
  memset(h, 0, sizeof *h);
  memcpy(h->magic, RD_FILE_MAGIC, 8);
  h->version = RD_FILE_VERSION;
  h->n = n;
  h->d = d;
  h->nlist = nlist;
  h->off_list_offsets = RD_FILE_ALIGN;
  h->off_ids = rd_fmt_align(h->off_list_offsets + 8ull * (uint64_t)(nlist + 1));
  h->off_centroids = rd_fmt_align(h->off_ids + 8ull * (uint64_t)n);
  h->off_vectors = rd_fmt_align(h->off_centroids + 4ull * (uint64_t)nlist * (uint64_t)d);
  h->file_bytes = h->off_vectors + 4ull * (uint64_t)n * (uint64_t)d;
}

static inline uint64_t rd_fmt_check(const rd_file_header* h, const int64_t* list_offsets) {
  uint64_t c = rd_fmt_fnv1a(0xcbf29ce484222325ull, h, (uint64_t)offsetof(rd_file_header, check));
  return rd_fmt_fnv1a(c, list_offsets, 8ull * (uint64_t)(h->nlist + 1));
}

/* 0 if the header is a well-formed v1 header for a file of file_bytes bytes, else a
 * static message describing the first problem. list_offsets may be NULL (header only). */
static inline const char* rd_fmt_validate(const rd_file_header* h, uint64_t file_bytes,
                                          const int64_t* list_offsets) {
  rd_file_header ref;
  if (memcmp(h->magic, RD_FILE_MAGIC, 8) != 0) return "not an rd index file (bad magic)";
  if (h->version != RD_FILE_VERSION) return "unsupported rd index file version";
  if (h->n < 0 || h->d < 1 || h->d > 65536 || h->nlist < 1) return "corrupt header (n, d, nlist)";
  rd_fmt_layout(&ref, h->n, h->d, h->nlist);
  if (ref.off_list_offsets != h->off_list_offsets || ref.off_ids != h->off_ids ||
      ref.off_centroids != h->off_centroids || ref.off_vectors != h->off_vectors ||
      ref.file_bytes != h->file_bytes)
    return "corrupt header (section offsets)";
  if (file_bytes < h->file_bytes) return "truncated rd index file";
  if (list_offsets) {
    if (rd_fmt_check(h, list_offsets) != h->check) return "rd index file checksum mismatch";
    if (list_offsets[0] != 0 || list_offsets[h->nlist] != h->n) return "corrupt list offsets";
    for (int32_t l = 0; l < h->nlist; ++l)
      if (list_offsets[l + 1] < list_offsets[l]) return "corrupt list offsets (not monotone)";
  }
  return 0;
}

#endif /* RD_FORMAT_H_ */
