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

#include <sys/stat.h>

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

// Streaming writer: sections go straight to the file (no whole-file buffer;
// a 1B-vector index is ~44 GB).
struct Writer {
    FILE* f = nullptr;
    std::string path;
    explicit Writer(const char* p) : path(p) {
        f = std::fopen(p, "wb");
        if (!f) throw IoError(std::string("cannot open file for writing: ") + p);
        std::setvbuf(f, nullptr, _IOFBF, 1 << 22);
    }
    ~Writer() {
        if (f) std::fclose(f);
    }
    void put(const void* p, size_t n) {
        if (n && std::fwrite(p, 1, n, f) != n) throw IoError("write failed: " + path);
    }
    template <class T>
    void pod(T v) { put(&v, sizeof(T)); }
    void close() {
        const int c = std::fclose(f);
        f = nullptr;
        if (c != 0) throw IoError("write failed: " + path);
    }
};

// Streaming reader: the file size comes from fstat and every section is read
// straight into its destination array.
struct Reader {
    FILE* f = nullptr;
    uint64_t size = 0, pos = 0;
    explicit Reader(const char* path) {
        f = std::fopen(path, "rb");
        if (!f) throw IoError(std::string("cannot open file: ") + path);
        struct stat st;
        if (fstat(fileno(f), &st) != 0) throw IoError(std::string("cannot stat file: ") + path);
        size = (uint64_t)st.st_size;
        std::setvbuf(f, nullptr, _IOFBF, 1 << 22);
    }
    ~Reader() {
        if (f) std::fclose(f);
    }
    uint64_t left() const { return size - pos; }
    void read(void* dst, uint64_t n) {
        if (n > left()) throw Corrupt();
        if (n && std::fread(dst, 1, n, f) != n) throw Corrupt();
        pos += n;
    }
    template <class T>
    T pod() {
        T v;
        read(&v, sizeof(T));
        return v;
    }
    void rewind() {
        std::fseek(f, 0, SEEK_SET);
        pos = 0;
    }
    void end() const {
        if (left()) throw Corrupt();
    }
};

struct QBlock {
    uint32_t d = 0, m = 0, ks = 0;
    std::vector<float> books;  // m * ks * (d / m) floats
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
    char mg[4];
    r.read(mg, 4);
    if (std::memcmp(mg, kMagic, 4) != 0) throw Corrupt();
    if (r.pod<uint8_t>() != kVersion) throw Corrupt();
    QBlock q;
    q.d = r.pod<uint32_t>();
    q.m = r.pod<uint32_t>();
    q.ks = r.pod<uint32_t>();
    if (q.d == 0 || q.m == 0 || q.ks == 0 || q.d % q.m) throw Corrupt();
    if ((uint64_t)q.ks * q.d * 4 > r.left()) throw Corrupt();
    q.books.resize((size_t)q.ks * q.d);
    r.read(q.books.data(), q.books.size() * 4);
    return q;
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

// pos_by_rank[r] = list position of the r-th smallest id.  Ids that form a
// dense range (every id-range shard written by this library) take a direct
// scatter (4 B per entry); anything else is sorted.  Duplicate ids are
// "corrupt file" (the partition invariant, ivf_index.hpp:27-36).
std::vector<uint32_t> pos_by_rank(const std::vector<uint32_t>& ids) {
    const size_t n = ids.size();
    std::vector<uint32_t> out(n);
    if (!n) return out;
    uint32_t lo = ids[0], hi = ids[0];
    for (uint32_t v : ids) {
        lo = std::min(lo, v);
        hi = std::max(hi, v);
    }
    if ((uint64_t)hi - lo + 1 == n) {
        std::vector<uint8_t> seen(n, 0);
        for (size_t i = 0; i < n; ++i) {
            const uint32_t r = ids[i] - lo;
            if (seen[r]) throw Corrupt();
            seen[r] = 1;
            out[r] = (uint32_t)i;
        }
        return out;
    }
    std::vector<uint64_t> ord(n);
    for (size_t i = 0; i < n; ++i) ord[i] = ((uint64_t)ids[i] << 32) | i;
    std::sort(ord.begin(), ord.end());
    for (size_t k = 0; k < n; ++k) {
        if (k && (ord[k] >> 32) == (ord[k - 1] >> 32)) throw Corrupt();  // duplicate id
        out[k] = (uint32_t)(ord[k] & 0xffffffffu);
    }
    return out;
}

// Parsed index file, lists in file order (ids ascending per list).
struct IndexFile {
    QBlock pq;
    uint32_t c = 0;
    std::vector<float> coarse;
    std::vector<uint64_t> offsets;  // c + 1
    std::vector<uint32_t> ids;      // list order
    std::vector<uint8_t> codes;     // list order
    bool refine = false;
    QBlock rq;
    std::vector<uint8_t> rcodes;    // list order
    uint64_t n = 0;
};

// Optional refinement section: refine quantizer block, m' u32, n*m' bytes in
// ascending id order, scattered to list order as it streams in.
void get_rblock(Reader& r, IndexFile& f, bool id_is_pos) {
    if (r.left() == 0) return;
    f.refine = true;
    f.rq = get_qblock(r);
    if (f.rq.d != f.pq.d || f.rq.ks > 256) throw Corrupt();
    const uint32_t mp = f.rq.m;
    if (r.pod<uint32_t>() != mp) throw Corrupt();
    if (f.n * mp > r.left()) throw Corrupt();
    f.rcodes.resize(f.n * mp);
    if (id_is_pos) {
        r.read(f.rcodes.data(), f.rcodes.size());
        return;
    }
    const std::vector<uint32_t> pbr = pos_by_rank(f.ids);
    constexpr size_t CH = 1 << 16;
    std::vector<uint8_t> buf(CH * mp);
    for (uint64_t k0 = 0; k0 < f.n; k0 += CH) {
        const size_t nk = (size_t)std::min<uint64_t>(CH, f.n - k0);
        r.read(buf.data(), nk * mp);
        for (size_t k = 0; k < nk; ++k)
            std::memcpy(&f.rcodes[(size_t)pbr[k0 + k] * mp], &buf[k * mp], mp);
    }
}

void parse_adc(Reader& r, IndexFile& f) {
    f.pq = get_qblock(r);
    if (f.pq.ks > 256) throw Corrupt();
    f.n = r.pod<uint64_t>();
    if (f.n > 0xffffffffull || f.n * f.pq.m > r.left()) throw Corrupt();
    f.codes.resize(f.n * f.pq.m);
    r.read(f.codes.data(), f.codes.size());
    f.c = 1;
    f.coarse.assign(f.pq.d, 0.f);
    f.offsets = {0, f.n};
    f.ids.resize(f.n);
    for (uint64_t i = 0; i < f.n; ++i) f.ids[i] = (uint32_t)i;
    get_rblock(r, f, true);
    r.end();
}

void parse_ivf(Reader& r, IndexFile& f) {
    f.pq = get_qblock(r);
    if (f.pq.ks > 256) throw Corrupt();
    f.c = r.pod<uint32_t>();
    if (f.c == 0 || (uint64_t)f.c * f.pq.d * 4 > r.left()) throw Corrupt();
    f.coarse.resize((size_t)f.c * f.pq.d);
    r.read(f.coarse.data(), f.coarse.size() * 4);
    if ((uint64_t)f.c * 8 > r.left()) throw Corrupt();
    f.offsets.assign(f.c + 1, 0);
    for (uint32_t l = 0; l < f.c; ++l) {
        const uint64_t len = r.pod<uint64_t>();
        if (len > r.left()) throw Corrupt();
        f.offsets[l + 1] = f.offsets[l] + len;
    }
    f.n = f.offsets[f.c];
    const uint32_t m = f.pq.m;
    const size_t rec = 4 + m;
    if (f.n > 0xffffffffull || f.n * rec > r.left()) throw Corrupt();
    f.ids.resize(f.n);
    f.codes.resize(f.n * m);
    constexpr size_t CH = 1 << 16;
    std::vector<uint8_t> buf(CH * rec);
    for (uint64_t i0 = 0; i0 < f.n; i0 += CH) {
        const size_t ni = (size_t)std::min<uint64_t>(CH, f.n - i0);
        r.read(buf.data(), ni * rec);
        for (size_t i = 0; i < ni; ++i) {
            std::memcpy(&f.ids[i0 + i], &buf[i * rec], 4);
            std::memcpy(&f.codes[(i0 + i) * m], &buf[i * rec + 4], m);
        }
    }
    for (uint32_t l = 0; l < f.c; ++l)
        for (uint64_t i = f.offsets[l] + 1; i < f.offsets[l + 1]; ++i)
            if (f.ids[i] <= f.ids[i - 1]) throw Corrupt();  // ids ascending per list
    get_rblock(r, f, false);
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

// refinement section: codes of all entries in ascending id order (id-aligned
// when the ids are 0..n-1, refine.hpp:21-28), streamed in chunks
void put_rblock(Writer& w, const Exported& e, bool id_is_pos) {
    const uint32_t mp = e.info.mprime;
    if (!mp) return;
    put_qblock(w, e.info.d, mp, e.info.ks, e.rbooks.data());
    w.pod<uint32_t>(mp);
    if (id_is_pos) {
        w.put(e.rcodes.data(), e.rcodes.size());
        return;
    }
    const std::vector<uint32_t> pbr = pos_by_rank(e.ids);
    constexpr size_t CH = 1 << 16;
    std::vector<uint8_t> buf(CH * mp);
    for (size_t k0 = 0; k0 < pbr.size(); k0 += CH) {
        const size_t nk = std::min(CH, pbr.size() - k0);
        for (size_t k = 0; k < nk; ++k) std::memcpy(&buf[k * mp], &e.rcodes[(size_t)pbr[k0 + k] * mp], mp);
        w.put(buf.data(), nk * mp);
    }
}

void load_into(pqrr_dev_index* ix, const IndexFile& f) {
    ck(pqrr_dev_load_lists(ix, f.offsets.data(), f.ids.data(), f.codes.data(),
                           f.refine ? f.rcodes.data() : nullptr));
}

}  // namespace
}  // namespace pqrr_b200

using namespace pqrr_b200;

extern "C" {

int pqrr_dev_save_quantizer(const char* path, uint32_t d, uint32_t m, uint32_t ks,
                            const float* books) {
    return run([&] {
        if (m == 0 || d % m) throw ArgError("dimension not divisible");
        Writer w(path);
        put_qblock(w, d, m, ks, books);
        w.close();
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
        if (books) std::memcpy(books, q.books.data(), q.books.size() * 4);
    });
}

int pqrr_dev_save_index(pqrr_dev_index* ix, const char* path) {
    return run([&] {
        Exported e = export_index(ix);
        const auto& in = e.info;
        Writer w(path);
        put_qblock(w, in.d, in.m, in.ks, e.books.data());
        w.pod<uint32_t>(in.c);
        w.put(e.coarse.data(), e.coarse.size() * 4);
        for (uint32_t l = 0; l < in.c; ++l) w.pod<uint64_t>(e.offsets[l + 1] - e.offsets[l]);
        const size_t rec = 4 + in.m;
        constexpr size_t CH = 1 << 16;
        std::vector<uint8_t> buf(CH * rec);
        for (uint64_t i0 = 0; i0 < in.n; i0 += CH) {
            const size_t ni = (size_t)std::min<uint64_t>(CH, in.n - i0);
            for (size_t i = 0; i < ni; ++i) {
                std::memcpy(&buf[i * rec], &e.ids[i0 + i], 4);
                std::memcpy(&buf[i * rec + 4], &e.codes[(i0 + i) * in.m], in.m);
            }
            w.put(buf.data(), ni * rec);
        }
        put_rblock(w, e, false);
        w.close();
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
        Writer w(path);
        put_qblock(w, in.d, in.m, in.ks, e.books.data());
        w.pod<uint64_t>(in.n);
        w.put(e.codes.data(), e.codes.size());
        put_rblock(w, e, true);
        w.close();
    });
}

int pqrr_dev_load_index(int device, const char* path, pqrr_dev_index** out) {
    *out = nullptr;
    return run([&] {
        Reader r(path);
        IndexFile f;
        parse_ivf(r, f);
        if (f.refine && f.rq.ks != f.pq.ks) throw Corrupt();
        pqrr_dev_index* ix = nullptr;
        ck(pqrr_dev_index_create(device, f.pq.d, f.c, f.coarse.data(), f.pq.m, f.pq.books.data(),
                                 f.refine ? f.rq.m : 0, f.refine ? f.rq.books.data() : nullptr,
                                 f.pq.ks, &ix));
        std::unique_ptr<pqrr_dev_index, int (*)(pqrr_dev_index*)> g(ix, pqrr_dev_index_destroy);
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
        if (f.refine && f.rq.ks != f.pq.ks) throw Corrupt();
        pqrr_dev_index* ix = nullptr;
        ck(pqrr_dev_adc_index_create(device, f.pq.d, f.pq.m, f.pq.books.data(),
                                     f.refine ? f.rq.m : 0, f.refine ? f.rq.books.data() : nullptr,
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
        r.rewind();
        IndexFile g;
        parse_ivf(r, g);  // throws "corrupt file" when neither layout fits
        *kind = PQRR_INDEX_IVF;
    });
}

}  // extern "C"
