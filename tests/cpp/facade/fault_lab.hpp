// Reference header name -> the B200 facade (tests/cpp/facade/abft_facade.hpp).
#pragma once
#include "abft_facade.hpp"
