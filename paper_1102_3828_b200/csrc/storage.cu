// storage.cu — the "PQRR" binary container (storage.hpp:14-28, SPEC.md:131,
// 194, 275) for quantizers, codebooks and device-resident ADC / IVF indexes.
// Host code only, written against the public C ABI (export / create / load
// entry points), so a saved index round-trips through any device.
//
// Layout (little-endian throughout; our reading of storage.hpp:18-27, which
// has no body in the reference):
//   quantizer block : "PQRR", version u8 = 1, d u32, m u32, ks u32,
//                     m*ks*(d/m) f32 (sub-quantizer-major, centroid-major,
//                     component-minor)
//   codebook file   : quantizer block with m = 1 (d = dim, ks = k)
//   adc index file  : quantizer block, n u64, n*m code bytes (id order),
//                     optional [refine quantizer block, m' u32, n*m' bytes]
//   ivf index file  : quantizer block (residual PQ), c u32, c*d f32 coarse
//                     centroids, c x u64 list lengths, per list its entries
//                     (id u32, m code bytes) with ids ascending, optional
//                     refine block as above (codes in ascending id order)
// Every load checks the magic, version, shapes and that the payload ends
// exactly at the end of the file ("corrupt file" otherwise).
#include <algorithm>
#include <cstdio>
#include <functional>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/pqrr_dev.h"
#include "internal.h"

static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__, "PQRR files are little-endian");

namespace pqrr_b200 {
namespace {

constexpr char kMagic[4] = {'P', 'Q', 'R', 'R'};
constexpr uint8_t kVersion = 1;

struct Corrupt : ArgError {
    Corrupt() : ArgError("corrupt file") {}
};
struct IoError : std::runtime_error {
    explicit IoError(const std::string& s) : std::runtime_error(s) {}
};

struct Writer {
    std::vector<uint8_t> buf;
    void put(const void* p, size_t n) {
        const uint8_t* b = static_cast<const uint8_t*>(p);
        buf.insert(buf.end(), b, b + n);
    }
    template <class T>
    void pod(T v) { put(&v, sizeof(T)); }
    void flush(const char* path) {
        FILE* f = std::fopen(path, "wb");
        if (!f) throw IoError(std::string("cannot open file for writing: ") + path);
        const size_t w = buf.empty() ? 0 : std::fwrite(buf.data(), 1, buf.size(), f);
        const int c = std::fclose(f);
        if (w != buf.size() || c != 0) throw IoError(std::string("write failed: ") + path);
    }
};

struct Reader {
    std::vector<uint8_t> buf;
    size_t pos = 0;
    explicit Reader(const char* path) {
        FILE* f = std::fopen(path, "rb");
        if (!f) throw IoError(std::string("cannot open file: ") + path);
        uint8_t tmp[1 << 16];
        size_t r;
        while ((r = std::fread(tmp, 1, sizeof tmp, f)) > 0) buf.insert(buf.end(), tmp, tmp + r);
        std::fclose(f);
    }
    size_t left() const { return buf.size() - pos; }
    const uint8_t* take(size_t n) {
        if (n > left()) throw Corrupt();
        const uint8_t* p = buf.data() + pos;
        pos += n;
        return p;
    }
    template <class T>
    T pod() {
        T v;
        std::memcpy(&v, take(sizeof(T)), sizeof(T));
        return v;
    }
    void end() const {
        if (left()) throw Corrupt();
    }
};

struct QBlock {
    uint32_t d = 0, m = 0, ks = 0;
    const float* books = nullptr;  // points into the reader's buffer (unaligned-safe copy below)
    std::vector<float> copy() const {
        std::vector<float> v((size_t)ks * d);
        std::memcpy(v.data(), books, v.size() * 4);
        return v;
    }
};

void put_qblock(Writer& w, uint32_t d, uint32_t m, uint32_t ks, const float* books) {
    w.put(kMagic, 4);
    w.pod<uint8_t>(kVersion);
    w.pod(d);
    w.pod(m);
    w.pod(ks);
    w.put(books, (size_t)ks * d * 4);  // m * ks * (d / m) floats
}

QBlock get_qblock(Reader& r) {
    const uint8_t* mg = r.take(4);
    if (std::memcmp(mg, kMagic, 4) != 0) throw Corrupt();
    if (r.pod<uint8_t>() != kVersion) throw Corrupt();
    QBlock q;
    q.d = r.pod<uint32_t>();
    q.m = r.pod<uint32_t>();
    q.ks = r.pod<uint32_t>();
    if (q.d == 0 || q.m == 0 || q.ks == 0 || q.d % q.m) throw Corrupt();
    if ((uint64_t)q.ks * q.d * 4 > r.left()) throw Corrupt();
    q.books = reinterpret_cast<const float*>(r.take((size_t)q.ks * q.d * 4));
    return q;
}

// Optional refinement section: refine quantizer block, m' u32, n*m' bytes.
struct RBlock {
    bool present = false;
    QBlock q;
    const uint8_t* codes = nullptr;
};

RBlock get_rblock(Reader& r, uint64_t n, uint32_t d) {
    RBlock b;
    if (r.left() == 0) return b;
    b.present = true;
    b.q = get_qblock(r);
    if (b.q.d != d || b.q.ks > 256) throw Corrupt();
    if (r.pod<uint32_t>() != b.q.m) throw Corrupt();
    if (n * b.q.m > r.left()) throw Corrupt();
    b.codes = r.take((size_t)(n * b.q.m));
    return b;
}

void ck(int rc) {
    if (rc != PQRR_OK) throw std::runtime_error(pqrr_dev_last_error());
}

int run(const std::function<void()>& f) {
    try {
        f();
        return PQRR_OK;
    } catch (const ArgError& e) {
        return report_error(PQRR_EINVAL, e.what());
    } catch (const std::exception& e) {
        return report_error(PQRR_EINTERNAL, e.what());
    }
}

// Parsed index file (pointers into the reader's buffer).
struct IndexFile {
    QBlock pq;
    uint32_t c = 0;
    const float* coarse = nullptr;
    std::vector<uint64_t> offsets;  // c + 1
    std::vector<uint32_t> ids;      // list order
    std::vector<uint8_t> codes;     // list order
    RBlock rb;
    uint64_t n = 0;
};

void parse_adc(Reader& r, IndexFile& f) {
    f.pq = get_qblock(r);
    if (f.pq.ks > 256) throw Corrupt();
    f.n = r.pod<uint64_t>();
    if (f.n > 0xffffffffull || f.n * f.pq.m > r.left()) throw Corrupt();
    const uint8_t* codes = r.take((size_t)(f.n * f.pq.m));
    f.c = 1;
    f.offsets = {0, f.n};
    f.ids.resize(f.n);
    for (uint64_t i = 0; i < f.n; ++i) f.ids[i] = (uint32_t)i;
    f.codes.assign(codes, codes + f.n * f.pq.m);
    f.rb = get_rblock(r, f.n, f.pq.d);
    r.end();
}

void parse_ivf(Reader& r, IndexFile& f) {
    f.pq = get_qblock(r);
    if (f.pq.ks > 256) throw Corrupt();
    f.c = r.pod<uint32_t>();
    if (f.c == 0 || (uint64_t)f.c * f.pq.d * 4 > r.left()) throw Corrupt();
    f.coarse = reinterpret_cast<const float*>(r.take((size_t)f.c * f.pq.d * 4));
    if ((uint64_t)f.c * 8 > r.left()) throw Corrupt();
    f.offsets.assign(f.c + 1, 0);
    for (uint32_t l = 0; l < f.c; ++l) {
        const uint64_t len = r.pod<uint64_t>();
        if (len > r.left()) throw Corrupt();
        f.offsets[l + 1] = f.offsets[l] + len;
    }
    f.n = f.offsets[f.c];
    const size_t rec = 4 + f.pq.m;
    if (f.n > 0xffffffffull || f.n * rec > r.left()) throw Corrupt();
    f.ids.resize(f.n);
    f.codes.resize(f.n * f.pq.m);
    for (uint64_t i = 0; i < f.n; ++i) {
        const uint8_t* e = r.take(rec);
        std::memcpy(&f.ids[i], e, 4);
        std::memcpy(&f.codes[i * f.pq.m], e + 4, f.pq.m);
    }
    for (uint32_t l = 0; l < f.c; ++l)
        for (uint64_t i = f.offsets[l] + 1; i < f.offsets[l + 1]; ++i)
            if (f.ids[i] <= f.ids[i - 1]) throw Corrupt();  // ids ascending per list
    f.rb = get_rblock(r, f.n, f.pq.d);
    r.end();
}

// Index contents pulled from the device (lists id-ascending).
struct Exported {
    pqrr_dev_index_info info{};
    std::vector<float> coarse, books, rbooks;
    std::vector<uint64_t> offsets;
    std::vector<uint32_t> ids;
    std::vector<uint8_t> codes, rcodes;  // list order
};

Exported export_index(pqrr_dev_index* ix) {
    Exported e;
    ck(pqrr_dev_index_get_info(ix, &e.info));
    const auto& in = e.info;
    e.coarse.resize((size_t)in.c * in.d);
    e.books.resize((size_t)in.ks * in.d);
    e.rbooks.resize(in.mprime ? (size_t)in.ks * in.d : 0);
    ck(pqrr_dev_export_codebooks(ix, e.coarse.data(), e.books.data(),
                                 in.mprime ? e.rbooks.data() : nullptr));
    e.offsets.resize(in.c + 1);
    e.ids.resize(in.n);
    e.codes.resize(in.n * in.m);
    e.rcodes.resize(in.n * in.mprime);
    ck(pqrr_dev_export_lists(ix, e.offsets.data(), e.ids.data(), e.codes.data(),
                             in.mprime ? e.rcodes.data() : nullptr));
    return e;
}

// refinement codes of all entries in ascending id order (id-aligned when the
// ids are 0..n-1, refine.hpp:21-28)
std::vector<uint8_t> rcodes_by_id(const Exported& e) {
    const uint32_t mp = e.info.mprime;
    std::vector<uint64_t> ord(e.ids.size());
    for (size_t i = 0; i < ord.size(); ++i) ord[i] = ((uint64_t)e.ids[i] << 32) | i;
    std::sort(ord.begin(), ord.end());
    std::vector<uint8_t> out(e.ids.size() * mp);
    for (size_t k = 0; k < ord.size(); ++k)
        std::memcpy(&out[k * mp], &e.rcodes[(ord[k] & 0xffffffffu) * mp], mp);
    return out;
}

void put_rblock(Writer& w, const Exported& e) {
    if (!e.info.mprime) return;
    put_qblock(w, e.info.d, e.info.mprime, e.info.ks, e.rbooks.data());
    w.pod<uint32_t>(e.info.mprime);
    const auto rc = rcodes_by_id(e);
    w.put(rc.data(), rc.size());
}

// list-order refinement codes from the id-ordered file section
std::vector<uint8_t> rcodes_list_order(const IndexFile& f) {
    const uint32_t mp = f.rb.q.m;
    std::vector<uint64_t> ord(f.ids.size());
    for (size_t i = 0; i < ord.size(); ++i) ord[i] = ((uint64_t)f.ids[i] << 32) | i;
    std::sort(ord.begin(), ord.end());
    std::vector<uint8_t> out(f.ids.size() * mp);
    for (size_t k = 0; k < ord.size(); ++k) {
        if (k && (ord[k] >> 32) == (ord[k - 1] >> 32)) throw Corrupt();  // duplicate id
        std::memcpy(&out[(ord[k] & 0xffffffffu) * mp], f.rb.codes + k * mp, mp);
    }
    return out;
}

void load_into(pqrr_dev_index* ix, const IndexFile& f) {
    std::vector<uint8_t> rc;
    if (f.rb.present) rc = rcodes_list_order(f);
    ck(pqrr_dev_load_lists(ix, f.offsets.data(), f.ids.data(), f.codes.data(),
                           f.rb.present ? rc.data() : nullptr));
}

}  // namespace
}  // namespace pqrr_b200

using namespace pqrr_b200;

extern "C" {

int pqrr_dev_save_quantizer(const char* path, uint32_t d, uint32_t m, uint32_t ks,
                            const float* books) {
    return run([&] {
        if (m == 0 || d % m) throw ArgError("dimension not divisible");
        Writer w;
        put_qblock(w, d, m, ks, books);
        w.flush(path);
    });
}

int pqrr_dev_load_quantizer(const char* path, uint32_t* d, uint32_t* m, uint32_t* ks,
                            float* books) {
    return run([&] {
        Reader r(path);
        QBlock q = get_qblock(r);
        r.end();
        *d = q.d;
        *m = q.m;
        *ks = q.ks;
        if (books) std::memcpy(books, q.books, (size_t)q.ks * q.d * 4);
    });
}

int pqrr_dev_save_index(pqrr_dev_index* ix, const char* path) {
    return run([&] {
        Exported e = export_index(ix);
        const auto& in = e.info;
        Writer w;
        put_qblock(w, in.d, in.m, in.ks, e.books.data());
        w.pod<uint32_t>(in.c);
        w.put(e.coarse.data(), e.coarse.size() * 4);
        for (uint32_t l = 0; l < in.c; ++l) w.pod<uint64_t>(e.offsets[l + 1] - e.offsets[l]);
        for (uint64_t i = 0; i < in.n; ++i) {
            w.pod<uint32_t>(e.ids[i]);
            w.put(&e.codes[i * in.m], in.m);
        }
        put_rblock(w, e);
        w.flush(path);
    });
}

int pqrr_dev_save_adc_index(pqrr_dev_index* ix, const char* path) {
    return run([&] {
        Exported e = export_index(ix);
        const auto& in = e.info;
        if (in.c != 1) throw ArgError("not an ADC index (more than one coarse cell)");
        for (float v : e.coarse)
            if (v != 0.f) throw ArgError("not an ADC index (non-zero coarse centroid)");
        for (uint64_t i = 0; i < in.n; ++i)
            if (e.ids[i] != i) throw ArgError("ADC files hold ids 0..n-1");
        Writer w;
        put_qblock(w, in.d, in.m, in.ks, e.books.data());
        w.pod<uint64_t>(in.n);
        w.put(e.codes.data(), e.codes.size());
        put_rblock(w, e);
        w.flush(path);
    });
}

int pqrr_dev_load_index(int device, const char* path, pqrr_dev_index** out) {
    *out = nullptr;
    return run([&] {
        Reader r(path);
        IndexFile f;
        parse_ivf(r, f);
        pqrr_dev_index* ix = nullptr;
        std::vector<float> books = f.pq.copy(), rb = f.rb.present ? f.rb.q.copy() : std::vector<float>();
        std::vector<float> coarse((size_t)f.c * f.pq.d);
        std::memcpy(coarse.data(), f.coarse, coarse.size() * 4);
        ck(pqrr_dev_index_create(device, f.pq.d, f.c, coarse.data(), f.pq.m, books.data(),
                                 f.rb.present ? f.rb.q.m : 0, f.rb.present ? rb.data() : nullptr,
                                 f.pq.ks, &ix));
        std::unique_ptr<pqrr_dev_index, int (*)(pqrr_dev_index*)> g(ix, pqrr_dev_index_destroy);
        if (f.rb.present && f.rb.q.ks != f.pq.ks) throw Corrupt();
        load_into(ix, f);
        *out = g.release();
    });
}

int pqrr_dev_load_adc_index(int device, const char* path, pqrr_dev_index** out) {
    *out = nullptr;
    return run([&] {
        Reader r(path);
        IndexFile f;
        parse_adc(r, f);
        if (f.rb.present && f.rb.q.ks != f.pq.ks) throw Corrupt();
        pqrr_dev_index* ix = nullptr;
        std::vector<float> books = f.pq.copy(), rb = f.rb.present ? f.rb.q.copy() : std::vector<float>();
        ck(pqrr_dev_adc_index_create(device, f.pq.d, f.pq.m, books.data(),
                                     f.rb.present ? f.rb.q.m : 0, f.rb.present ? rb.data() : nullptr,
                                     f.pq.ks, &ix));
        std::unique_ptr<pqrr_dev_index, int (*)(pqrr_dev_index*)> g(ix, pqrr_dev_index_destroy);
        load_into(ix, f);
        *out = g.release();
    });
}

int pqrr_dev_probe_index_kind(const char* path, int* kind) {
    return run([&] {
        Reader r(path);
        IndexFile f;
        try {
            parse_adc(r, f);
            *kind = PQRR_INDEX_ADC;
            return;
        } catch (const Corrupt&) {
        }
        r.pos = 0;
        IndexFile g;
        parse_ivf(r, g);  // throws "corrupt file" when neither layout fits
        *kind = PQRR_INDEX_IVF;
    });
}

}  // extern "C"
