// shard_detail.h -- the shard header writer and validating parser behind
// fntrs::shardio::write_shard / read_shard (dropin_aux.cpp), shared with the
// batched file tool (cli.cpp), which converts whole payload matrices on the
// device instead of one shard at a time.
#pragma once
#include <cstdint>
#include <span>
#include <vector>

#include "fntrs/shardio.hpp"

namespace fntrs::shardio::detail {

// header + escape list of a shard with `symbols` payload words (the reference's
// write_shard checks, in order: k, n, index, length, escape count)
std::vector<std::uint8_t> shard_header(const ShardInfo& info, std::uint64_t symbols,
                                       const std::vector<std::uint64_t>& escapes);

struct ParsedShard {
    ShardInfo info;
    std::uint32_t symbols = 0;
    std::vector<std::uint32_t> escapes;  // ascending positions < symbols, all on zero words
    std::size_t payload_offset = 0;      // big-endian words start here
};

// read_shard's validation (every error class and order of the reference)
// without converting the payload.
ParsedShard parse_shard(std::span<const std::uint8_t> bytes);

}  // namespace fntrs::shardio::detail
