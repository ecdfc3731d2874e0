// QCNM model store (the reference's model file, src/model_store.cpp): a zero-copy
// reader over an mmap of the file and the matching writer.  Host code only.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "qnb_internal.h"

struct qnb_model {
  void* map = nullptr;
  size_t size = 0;
  std::vector<std::string> names;
  std::vector<qnb_record> recs;
};

namespace {

constexpr char kMagic[4] = {'Q', 'C', 'N', 'M'};
constexpr uint8_t kVersion = 1;

int64_t byte_width(int32_t dt) { return dt == QNB_FP32 ? 4 : (dt == QNB_INT8Q ? 1 : 2); }

// Little-endian cursor; every read checks the remaining length first.
struct Cursor {
  const uint8_t* p;
  size_t left;
  bool take(size_t n) {
    if (n > left) return false;
    left -= n;
    return true;
  }
  bool u8(uint8_t* v) {
    if (!take(1)) return false;
    *v = *p++;
    return true;
  }
  bool u16(uint16_t* v) {
    if (!take(2)) return false;
    *v = (uint16_t)(p[0] | (p[1] << 8));
    p += 2;
    return true;
  }
  bool u32(uint32_t* v) {
    if (!take(4)) return false;
    *v = (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
    p += 4;
    return true;
  }
  bool f32(float* v) {
    uint32_t b;
    if (!u32(&b)) return false;
    std::memcpy(v, &b, 4);
    return true;
  }
};

void put_u32(std::string* o, uint32_t v) {
  for (int i = 0; i < 4; ++i) o->push_back((char)((v >> (8 * i)) & 0xff));
}
void put_f32(std::string* o, float v) {
  uint32_t b;
  std::memcpy(&b, &v, 4);
  put_u32(o, b);
}

qnb_status parse(qnb_model* m) {
  const uint8_t* base = static_cast<const uint8_t*>(m->map);
  if (m->size < 9 || std::memcmp(base, kMagic, 4) != 0 || base[4] != kVersion)
    return qnb::fail(QNB_E_IO, "not a model file");
  Cursor c{base + 5, m->size - 5};
  const char* trunc = "truncated model file";
  uint32_t count;
  if (!c.u32(&count)) return qnb::fail(QNB_E_IO, trunc);
  // the count is untrusted: a record takes at least 31 bytes (name length, tag, rank,
  // six floats), so never reserve more than the rest of the file can hold
  const size_t fit = c.left / 31;
  m->names.reserve(std::min<size_t>(count, fit));
  m->recs.reserve(std::min<size_t>(count, fit));
  for (uint32_t i = 0; i < count; ++i) {
    qnb_record r;
    std::memset(&r, 0, sizeof(r));
    uint16_t len;
    if (!c.u16(&len)) return qnb::fail(QNB_E_IO, trunc);
    const uint8_t* np = c.p;
    if (!c.take(len)) return qnb::fail(QNB_E_IO, trunc);
    c.p += len;
    m->names.emplace_back(reinterpret_cast<const char*>(np), len);
    uint8_t tag, rank;
    if (!c.u8(&tag)) return qnb::fail(QNB_E_IO, trunc);
    if (tag > QNB_INT16Q) return qnb::fail(QNB_E_IO, "not a model file");
    r.dtype = tag;
    if (!c.u8(&rank)) return qnb::fail(QNB_E_IO, trunc);
    if (rank > 8) return qnb::fail(QNB_E_UNSUPPORTED, "model record of rank > 8: " + m->names.back());
    r.rank = rank;
    int64_t count_el = 1;  // shape_count: product of the extents (1 for rank 0)
    for (int d = 0; d < rank; ++d) {
      uint32_t e;
      if (!c.u32(&e)) return qnb::fail(QNB_E_IO, trunc);
      r.extents[d] = e;
      count_el *= (int64_t)e;
    }
    float reserved;
    if (!c.f32(&r.f_min) || !c.f32(&r.f_max) || !c.f32(&r.scale) || !c.f32(&r.zero) || !c.f32(&r.one) ||
        !c.f32(&reserved))
      return qnb::fail(QNB_E_IO, trunc);
    r.payload_bytes = count_el * byte_width(r.dtype);
    r.payload = c.p;
    if (!c.take((size_t)r.payload_bytes)) return qnb::fail(QNB_E_IO, trunc);
    c.p += r.payload_bytes;
    m->recs.push_back(r);
  }
  for (size_t i = 0; i < m->recs.size(); ++i) m->recs[i].name = m->names[i].c_str();
  return QNB_OK;
}

}  // namespace

extern "C" {

qnb_status qnb_model_open(const char* path, qnb_model** out) {
  return qnb::guarded([&]() -> qnb_status {
    if (!path || !out) return qnb::fail(QNB_E_ARG, "null argument");
    *out = nullptr;
    const int fd = ::open(path, O_RDONLY);
    if (fd < 0) return qnb::fail(QNB_E_IO, std::string("cannot read: ") + path);
    struct stat st;
    if (::fstat(fd, &st) != 0) {
      ::close(fd);
      return qnb::fail(QNB_E_IO, std::string("cannot read: ") + path);
    }
    auto* m = new qnb_model;
    m->size = (size_t)st.st_size;
    if (m->size > 0) {
      m->map = ::mmap(nullptr, m->size, PROT_READ, MAP_PRIVATE, fd, 0);
      if (m->map == MAP_FAILED) {
        m->map = nullptr;
        ::close(fd);
        delete m;
        return qnb::fail(QNB_E_IO, std::string("cannot read: ") + path);
      }
    }
    ::close(fd);
    const qnb_status s = parse(m);
    if (s != QNB_OK) {
      qnb_model_close(m);
      return s;
    }
    *out = m;
    return QNB_OK;
  });
}

qnb_status qnb_model_count(const qnb_model* m, int64_t* n) {
  if (!m || !n) return qnb::fail(QNB_E_ARG, "null argument");
  *n = (int64_t)m->recs.size();
  return QNB_OK;
}

qnb_status qnb_model_record(const qnb_model* m, int64_t i, qnb_record* out) {
  if (!m || !out) return qnb::fail(QNB_E_ARG, "null argument");
  if (i < 0 || i >= (int64_t)m->recs.size()) return qnb::fail(QNB_E_ARG, "record index out of range");
  *out = m->recs[(size_t)i];
  return QNB_OK;
}

qnb_status qnb_model_close(qnb_model* m) {
  if (!m) return QNB_OK;
  if (m->map) ::munmap(m->map, m->size);
  delete m;
  return QNB_OK;
}

qnb_status qnb_model_save(const char* path, const qnb_record* recs, int64_t n) {
  return qnb::guarded([&]() -> qnb_status {
    if (!path || (n > 0 && !recs) || n < 0) return qnb::fail(QNB_E_ARG, "null argument");
    std::string buf(kMagic, 4);
    buf.push_back((char)kVersion);
    put_u32(&buf, (uint32_t)n);
    for (int64_t i = 0; i < n; ++i) {
      const qnb_record& r = recs[i];
      const std::string name = r.name ? r.name : "";
      if (name.size() > 0xffff) return qnb::fail(QNB_E_ARG, "record name too long: " + name);
      if (r.rank < 0 || r.rank > 8 || r.dtype < QNB_FP32 || r.dtype > QNB_INT16Q)
        return qnb::fail(QNB_E_ARG, "invalid record: " + name);
      int64_t count_el = 1;
      for (int d = 0; d < r.rank; ++d) count_el *= r.extents[d];
      if (r.payload_bytes != count_el * byte_width(r.dtype) || (r.payload_bytes > 0 && !r.payload))
        return qnb::fail(QNB_E_ARG, "payload size mismatch: " + name);
      buf.push_back((char)(name.size() & 0xff));
      buf.push_back((char)((name.size() >> 8) & 0xff));
      buf.append(name);
      buf.push_back((char)(uint8_t)r.dtype);
      buf.push_back((char)(uint8_t)r.rank);
      for (int d = 0; d < r.rank; ++d) put_u32(&buf, (uint32_t)r.extents[d]);
      put_f32(&buf, r.f_min);
      put_f32(&buf, r.f_max);
      put_f32(&buf, r.scale);
      put_f32(&buf, r.zero);
      put_f32(&buf, r.one);
      put_f32(&buf, 0.0f);  // reserved
      buf.append(static_cast<const char*>(r.payload), (size_t)r.payload_bytes);
    }
    const std::string tmp = std::string(path) + ".tmp";
    FILE* f = std::fopen(tmp.c_str(), "wb");
    if (!f) return qnb::fail(QNB_E_IO, "cannot write: " + tmp);
    const bool ok = std::fwrite(buf.data(), 1, buf.size(), f) == buf.size();
    if (std::fclose(f) != 0 || !ok) return qnb::fail(QNB_E_IO, "cannot write: " + tmp);
    if (std::rename(tmp.c_str(), path) != 0) return qnb::fail(QNB_E_IO, std::string("cannot write: ") + path);
    return QNB_OK;
  });
}

}  // extern "C"
