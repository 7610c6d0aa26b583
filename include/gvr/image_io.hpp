// gvr/image_io.hpp — the reference's image formats (proj/include/gvr/image_io.hpp,
// src/image_io.cpp) for the C++ drop-in: PFM read / write, PNG write. Host file
// I/O only (no compute). PNG input needs an inflater, which this image lacks
// (no libpng / zlib): read_png reports that; PFM is the lossless path anyway.
#pragma once

#include "gvr.hpp"

#include <cstdio>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

namespace gvr {

namespace detail {

inline void write_file_atomic(const std::filesystem::path& path, const std::string& bytes) {
    std::filesystem::path tmp = path;
    tmp += ".tmp";
    {
        std::ofstream out(tmp, std::ios::binary | std::ios::trunc);
        if (!out) throw ValidationError("cannot write file: " + tmp.string());
        out.write(bytes.data(), static_cast<std::streamsize>(bytes.size()));
        if (!out) throw ValidationError("write failed: " + tmp.string());
    }
    std::error_code ec;
    std::filesystem::rename(tmp, path, ec);
    if (ec) throw ValidationError("cannot move temp file onto " + path.string() + ": " + ec.message());
}

inline uint32_t crc32_png(const unsigned char* p, size_t n, uint32_t c = 0xffffffffu) {
    for (size_t i = 0; i < n; ++i) {
        c ^= p[i];
        for (int k = 0; k < 8; ++k) c = (c >> 1) ^ (0xedb88320u & (0u - (c & 1u)));
    }
    return c;
}

inline void put_be32(std::string& s, uint32_t v) {
    for (int i = 3; i >= 0; --i) s.push_back(static_cast<char>((v >> (8 * i)) & 0xff));
}

inline void png_chunk(std::string& out, const char* type, const std::string& data) {
    put_be32(out, static_cast<uint32_t>(data.size()));
    std::string td(type, 4);
    td += data;
    out += td;
    put_be32(out, crc32_png(reinterpret_cast<const unsigned char*>(td.data()), td.size()) ^ 0xffffffffu);
}

}  // namespace detail

// image_io.cpp:35-75: 8-bit PNG, value = lround(clamp(v, 0, 1) * 255), 1 or 3 channels.
// The image data is stored in uncompressed deflate blocks (valid PNG; no zlib here).
inline void write_png(const Image& image, const std::filesystem::path& path) {
    if (image.channels != 1 && image.channels != 3) throw ValidationError("write_png supports 1 or 3 channels");
    std::string raw;
    for (int i = 0; i < image.height; ++i) {
        raw.push_back('\0');  // filter: none
        for (int j = 0; j < image.width; ++j)
            for (int c = 0; c < image.channels; ++c) {
                const double v = std::clamp(image.at(i, j, c), 0.0, 1.0);
                raw.push_back(static_cast<char>(static_cast<unsigned char>(std::lround(v * 255.0))));
            }
    }
    std::string z = "\x78\x01";  // zlib header, no compression
    uint32_t a = 1, b = 0;
    for (unsigned char ch : raw) {
        a = (a + ch) % 65521u;
        b = (b + a) % 65521u;
    }
    for (size_t pos = 0; pos < raw.size() || pos == 0; pos += 65535) {
        const size_t len = std::min<size_t>(65535, raw.size() - pos);
        z.push_back(pos + len >= raw.size() ? '\x01' : '\x00');
        z.push_back(static_cast<char>(len & 0xff));
        z.push_back(static_cast<char>(len >> 8));
        z.push_back(static_cast<char>(~len & 0xff));
        z.push_back(static_cast<char>((~len >> 8) & 0xff));
        z.append(raw, pos, len);
        if (raw.empty()) break;
    }
    detail::put_be32(z, (b << 16) | a);
    std::string out("\x89PNG\r\n\x1a\n", 8), ihdr;
    detail::put_be32(ihdr, static_cast<uint32_t>(image.width));
    detail::put_be32(ihdr, static_cast<uint32_t>(image.height));
    ihdr += std::string("\x08", 1) + (image.channels == 3 ? std::string("\x02", 1) : std::string("\x00", 1)) +
            std::string("\x00\x00\x00", 3);
    detail::png_chunk(out, "IHDR", ihdr);
    detail::png_chunk(out, "IDAT", z);
    detail::png_chunk(out, "IEND", "");
    detail::write_file_atomic(path, out);
}

// image_io.cpp:77-122
inline Image read_png(const std::filesystem::path& path) {
    throw ValidationError("cannot read PNG " + path.string() + ": no PNG decoder in this build (use PFM)");
}

// image_io.cpp:124-157: "PF" (3 channels) / "Pf" (1 channel), little-endian
// (scale -1.0), rows bottom-up, float32.
inline void write_pfm(const Image& image, const std::filesystem::path& path) {
    if (image.channels != 1 && image.channels != 3) throw ValidationError("write_pfm supports 1 or 3 channels");
    std::ostringstream head;
    head << (image.channels == 3 ? "PF" : "Pf") << "\n" << image.width << " " << image.height << "\n-1.0\n";
    std::string out = head.str();
    for (int i = image.height - 1; i >= 0; --i)
        for (int j = 0; j < image.width; ++j)
            for (int c = 0; c < image.channels; ++c) {
                const float v = static_cast<float>(image.at(i, j, c));
                char b[4];
                std::memcpy(b, &v, 4);  // little-endian host
                out.append(b, 4);
            }
    detail::write_file_atomic(path, out);
}

// image_io.cpp:159-190
inline Image read_pfm(const std::filesystem::path& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw ValidationError("cannot open file: " + path.string());
    std::string magic;
    int w = 0, h = 0;
    double scale = 0.0;
    if (!(in >> magic >> w >> h >> scale) || (magic != "PF" && magic != "Pf") || w <= 0 || h <= 0)
        throw ValidationError("not a PFM file: " + path.string());
    if (scale >= 0.0) throw ValidationError("big-endian PFM is not supported: " + path.string());
    in.get();  // the single whitespace after the scale
    const int ch = magic == "PF" ? 3 : 1;
    std::vector<float> buf(static_cast<size_t>(w) * h * ch);
    in.read(reinterpret_cast<char*>(buf.data()), static_cast<std::streamsize>(buf.size() * 4));
    if (in.gcount() != static_cast<std::streamsize>(buf.size() * 4))
        throw ValidationError("truncated PFM data: " + path.string());
    Image img(h, w, ch, ch == 3 ? ChannelSemantics::Color : ChannelSemantics::Feature);
    for (int i = 0; i < h; ++i)
        for (int j = 0; j < w; ++j)
            for (int c = 0; c < ch; ++c)
                img.at(h - 1 - i, j, c) = buf[(static_cast<size_t>(i) * w + j) * ch + c];
    return img;
}

}  // namespace gvr
